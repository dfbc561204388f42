"""Host setup of the tau (sine-transform) preconditioner of the implicit-step operator.

For the orthonormal DST-I matrices S_x, S_y (orders nx, ny) the optimal
Frobenius-norm approximation of A = M + s (Kx A_x + Ky A_y) in the 2-D tau
algebra {(S_y (x) S_x) diag(d) (S_y (x) S_x)} has

    d = diag((S_y (x) S_x) A (S_y (x) S_x)) = D_m + s * D_k.

Every operator here is a sum of Kronecker products E (x) T of a y-factor and an
x-factor (I, the shift U, U^T against Toeplitz blocks, assembly.py:100-128), so
d is a sum of outer products diag(S_y E S_y) diag(S_x T S_x)^T: O(n^3) setup on
the host, done once per grid.  A is SPD, hence d > 0 and P = (S(x)S) diag(d) (S(x)S)
is SPD.  P^{-1} is applied on the device as four dense DST contractions (DMMA)
plus a diagonal scaling.  The preconditioner changes only the inner-solve
iteration count: every solve still stops on the reference criterion
||b - A x|| <= rel_tol ||b|| (krylov.py:48-83), so MGRIT results stay within
the parity tolerance.
"""

from __future__ import annotations

import numpy as np

__all__ = ["dst_matrix", "tau_diagonals", "tau_diagonals_from_generators"]


def dst_matrix(n: int) -> np.ndarray:
    k = np.arange(1, n + 1)
    return np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(k, k) / (n + 1))


def _sts(S: np.ndarray, T: np.ndarray) -> np.ndarray:
    """diag(S T S) through one GEMM (S symmetric): O(n^3) on the BLAS, 1023^2 grids in well under a second."""
    return np.einsum("ij,ij->i", S @ T, S)


def _toeplitz(col, row):
    from scipy.linalg import toeplitz

    return toeplitz(np.asarray(col, dtype=float), np.asarray(row, dtype=float))


def tau_diagonals_from_generators(gens, nx: int, ny: int, kx: float, ky: float):
    """(D_m, D_k) from an engine's generator set (engine.Generators); P1 mass stencil assumed."""
    Sx, Sy = dst_matrix(nx), dst_matrix(ny)
    ex = _sts(Sx, np.eye(nx, k=1))
    ey = _sts(Sy, np.eye(ny, k=1))
    m1 = np.zeros(nx)
    m1[: min(nx, 2)] = [6.0, 1.0][: min(nx, 2)]
    m2c = np.zeros(nx)
    m2c[0] = 1.0
    m2r = m2c.copy()
    if nx > 1:
        m2r[1] = 1.0
    dm = gens.mass_scale * (np.outer(np.ones(ny), _sts(Sx, _toeplitz(m1, m1)))
                            + 2.0 * np.outer(ey, _sts(Sx, _toeplitz(m2c, m2r))))
    dx = gens.sx * (np.outer(np.ones(ny), _sts(Sx, _toeplitz(gens.t1x_col, gens.t1x_row)))
                    + 2.0 * np.outer(ey, _sts(Sx, _toeplitz(gens.t2x_col, gens.t2x_row))))
    dy = gens.sy * (np.outer(_sts(Sy, _toeplitz(gens.t1y_col, gens.t1y_row)), np.ones(nx))
                    + 2.0 * np.outer(_sts(Sy, _toeplitz(gens.t2y_col, gens.t2y_row)), ex))
    return dm, kx * dx + ky * dy


def tau_diagonals(grid, beta: float, gamma: float, kx: float, ky: float):
    """(D_m, D_k) as [ny, nx] arrays: d(s) = D_m + s * D_k for the operator M + s (Kx Ax + Ky Ay)."""
    from .assembly import mass_generators, stiffness_generators, stiffness_scale

    nx, ny = grid.nx, grid.ny
    Sx, Sy = dst_matrix(nx), dst_matrix(ny)
    # diag(S U S) for the one-step shift (identical for U^T); the identity gives ones
    ex = _sts(Sx, np.eye(nx, k=1))
    ey = _sts(Sy, np.eye(ny, k=1))
    m1, m2, cm = mass_generators(grid)
    a1x, a2x = stiffness_generators(grid.mx, beta)
    a1y, a2y = stiffness_generators(grid.my, gamma)
    sx = stiffness_scale(grid.hx, grid.hy, beta)
    sy = stiffness_scale(grid.hy, grid.hx, gamma)
    # x-axis operators: scale * (I (x) T1 + U (x) T2 + U^T (x) T2^T), (y-factor) (x) (x-factor)
    dm = cm * (np.outer(np.ones(ny), _sts(Sx, m1.dense)) + 2.0 * np.outer(ey, _sts(Sx, m2.dense)))
    dx = sx * (np.outer(np.ones(ny), _sts(Sx, a1x.dense)) + 2.0 * np.outer(ey, _sts(Sx, a2x.dense)))
    # y-axis operator: scale * (T1 (x) I + T2 (x) U + T2^T (x) U^T)
    dy = sy * (np.outer(_sts(Sy, a1y.dense), np.ones(nx)) + 2.0 * np.outer(_sts(Sy, a2y.dense), ex))
    return dm, kx * dx + ky * dy
