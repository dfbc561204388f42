"""Mass and fractional-stiffness operators (mirrors riesz_mgrit/assembly.py).

The generators are closed forms evaluated on the host (O(n), setup only).
``apply`` runs on the B200: the block-tridiagonal-Toeplitz matvec is the DMMA
kernel of csrc/rm_device.cuh, fed from the O(n) generator tables (the dense
Toeplitz blocks of the reference, assembly.py:58-60, are never formed on the
device).  ``dense`` (host, capped) exists for the small dense-oracle checks the
reference also offers (assembly.py:117-128).

``apply`` accepts a vector ``[ndof]``, a batch ``[B, ndof]`` (numpy or a
float64 CUDA tensor) and returns the same kind.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch
from scipy.linalg import toeplitz

from .krylov import CgOptions
from .mesh import SpatialGrid

__all__ = [
    "ToeplitzGenerator",
    "BttbOperator",
    "CombinedStepOperator",
    "mass_generators",
    "stiffness_generators",
    "stiffness_scale",
    "mass_operator",
    "stiffness_operator_x",
    "stiffness_operator_y",
    "combined_step_operator",
    "dense_instantiation",
    "permutation_to_column_major",
    "DENSE_CAP",
]

DENSE_CAP = 4096


@dataclass(frozen=True)
class ToeplitzGenerator:
    """First column and first row of a square Toeplitz block (assembly.py:37-60)."""

    first_col: np.ndarray
    first_row: np.ndarray

    def __post_init__(self):
        col = np.asarray(self.first_col, dtype=float)
        row = np.asarray(self.first_row, dtype=float)
        if col.size != row.size:
            raise ValueError("column and row lengths differ")
        if col[0] != row[0]:
            raise ValueError("corner entries disagree")
        object.__setattr__(self, "first_col", col)
        object.__setattr__(self, "first_row", row)

    @property
    def size(self) -> int:
        return self.first_col.size

    @cached_property
    def dense(self) -> np.ndarray:
        return toeplitz(self.first_col, self.first_row)


# ----------------------------------------------------------------------------
# closed-form generators (assembly.py:172-251)
# ----------------------------------------------------------------------------


def mass_generators(grid: SpatialGrid):
    """(M1, M2, hx*hy/12): M1 = tridiag(1, 6, 1), M2 = upper bidiagonal (1, 1)."""
    n = grid.mx - 1
    m1 = np.zeros(n)
    m1[:2] = [6.0, 1.0][: min(n, 2)]
    c2 = np.zeros(n)
    c2[0] = 1.0
    r2 = c2.copy()
    if n > 1:
        r2[1] = 1.0
    return ToeplitzGenerator(m1, m1.copy()), ToeplitzGenerator(c2, r2), grid.hx * grid.hy / 12.0


def _power_sums(l: np.ndarray, e: float):
    return {k: np.abs(l + k) ** e for k in (-2, -1, 0, 1, 2)}


def stiffness_generators(M: int, rho: float):
    """Generators (A1, A2) of the 1-D fractional stiffness blocks, prefactor excluded.

    A1 is symmetric; A2's first row starts (d, d, ...) and its first column is
    the row formula shifted by one (assembly.py:226-249).
    """
    if not 0.5 < rho < 1.0:
        raise ValueError("fractional half-order must lie in (1/2, 1)")
    if M < 2:
        raise ValueError("need at least 2 intervals")
    n = M - 1
    p3, p4 = 3.0 - 2.0 * rho, 4.0 - 2.0 * rho
    head1 = [2.0 ** (6.0 - 2.0 * rho) + 16.0 * rho - 40.0,
             2.0 * 3.0**p4 + (2.0 * rho - 6.0) * 2.0 ** (5.0 - 2.0 * rho) - 16.0 * rho + 34.0]
    a1 = np.zeros(n)
    a1[: min(n, 2)] = head1[: min(n, 2)]
    if n > 2:
        l = np.arange(2.0, n)
        q = _power_sums(l, p3)
        w = _power_sums(l, p4)
        a1[2:] = (4.0 * p4 * (-q[-1] + 2.0 * q[0] - q[1])
                  - 2.0 * w[-2] + 4.0 * w[-1] - 4.0 * w[1] + 2.0 * w[2])
    diag = 4.0 - 2.0**p4 * rho
    row = np.zeros(n)
    col = np.zeros(n)
    row[0] = col[0] = diag
    if n > 1:
        row[1] = diag
    if n > 2:
        l = np.arange(2.0, n)
        q = _power_sums(l, p3)
        w = _power_sums(l, p4)
        row[2:] = (p4 * (q[-2] - q[-1] - q[0] + q[1])
                   + 2.0 * w[-2] - 6.0 * w[-1] + 6.0 * w[0] - 2.0 * w[1])
    if n > 1:
        m = np.arange(1.0, n)
        q = _power_sums(m, p3)
        w = _power_sums(m, p4)
        col[1:] = (p4 * (q[-1] - q[0] - q[1] + q[2])
                   + 2.0 * w[-1] - 6.0 * w[0] + 6.0 * w[1] - 2.0 * w[2])
    return ToeplitzGenerator(a1, a1.copy()), ToeplitzGenerator(col, row)


def stiffness_scale(h_along: float, h_across: float, rho: float) -> float:
    """h^{1-2rho} h' / (2 cos(rho pi) Gamma(5 - 2rho))  (assembly.py:259-274); negative on (1/2, 1)."""
    return h_along ** (1.0 - 2.0 * rho) * h_across / (2.0 * math.cos(rho * math.pi) * math.gamma(5.0 - 2.0 * rho))


# ----------------------------------------------------------------------------
# array plumbing (numpy <-> device)
# ----------------------------------------------------------------------------


def to_device_2d(v, ndof: int):
    """Return (tensor [B, ndof] on the device, kind) where kind records the caller's type/shape."""
    from .engine import require_cuda

    dev = require_cuda()
    if isinstance(v, torch.Tensor):
        t = v.to(device=dev, dtype=torch.float64)
        kind = ("torch", tuple(v.shape))
    else:
        a = np.asarray(v, dtype=float)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        kind = ("numpy", a.shape)
    if t.numel() % ndof or t.shape[-1] != ndof:
        raise ValueError(f"expected vector of length {ndof}, got {tuple(t.shape)}")
    return t.reshape(-1, ndof).contiguous(), kind


def from_device(t: torch.Tensor, kind):
    typ, shape = kind
    if typ == "torch":
        return t.reshape(shape)
    return t.reshape(shape).cpu().numpy()


# ----------------------------------------------------------------------------
# operators
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class BttbOperator:
    """scale * block-tridiagonal operator with Toeplitz blocks (assembly.py:63-128)."""

    scale: float
    diag_block: ToeplitzGenerator
    off_block: ToeplitzGenerator
    axis: str
    block_count: int

    def __post_init__(self):
        if self.axis not in ("x", "y"):
            raise ValueError("axis must be 'x' or 'y'")

    @property
    def block_size(self) -> int:
        return self.diag_block.size

    @property
    def ndof(self) -> int:
        return self.block_size * self.block_count

    @property
    def grid_shape(self) -> tuple[int, int]:
        """(ny, nx), x fastest."""
        if self.axis == "x":
            return (self.block_count, self.block_size)
        return (self.block_size, self.block_count)

    @cached_property
    def _engine(self):
        from .engine import Engine, Generators

        ny, nx = self.grid_shape
        z = lambda k: np.zeros(k)  # noqa: E731
        d, o = self.diag_block, self.off_block
        if self.axis == "x":
            gens = Generators(d.first_col, d.first_row, o.first_col, o.first_row, z(ny), z(ny), z(ny), z(ny),
                              self.scale, 0.0, 0.0)
        else:
            gens = Generators(z(nx), z(nx), z(nx), z(nx), d.first_col, d.first_row, o.first_col, o.first_row,
                              0.0, self.scale, 0.0)
        return Engine(nx, ny, gens, 1.0, 1.0)

    def apply(self, v):
        t, kind = to_device_2d(v, self.ndof)
        return from_device(self._engine.apply(2 if self.axis == "x" else 3, t), kind)

    def dense(self, cap: int = DENSE_CAP) -> np.ndarray:
        if self.ndof > cap:
            raise ValueError(f"dense instantiation of order {self.ndof} exceeds cap {cap}")
        T1, T2 = self.diag_block.dense, self.off_block.dense
        n = self.block_count
        sup = np.eye(n, k=1)
        if self.axis == "x":
            full = np.kron(np.eye(n), T1) + np.kron(sup, T2) + np.kron(sup.T, T2.T)
        else:
            full = np.kron(T1, np.eye(n)) + np.kron(T2, sup) + np.kron(T2.T, sup.T)
        return self.scale * full


def _is_standard_mass(op: BttbOperator) -> bool:
    n = op.block_size
    m1, m2, _ = mass_generators(SpatialGrid(n + 1, 2))
    return (op.axis == "x" and np.array_equal(op.diag_block.first_col, m1.first_col)
            and np.array_equal(op.diag_block.first_row, m1.first_row)
            and np.array_equal(op.off_block.first_col, m2.first_col)
            and np.array_equal(op.off_block.first_row, m2.first_row))


@dataclass(frozen=True)
class CombinedStepOperator:
    """mass + sign * half_dt * (kx * stiff_x + ky * stiff_y) (assembly.py:131-169)."""

    mass: BttbOperator
    stiff_x: BttbOperator
    stiff_y: BttbOperator
    kx: float
    ky: float
    half_dt: float
    sign: int
    engine: object = None  # shared device context (set by Discretization)

    def __post_init__(self):
        if self.sign not in (+1, -1):
            raise ValueError("sign must be +1 or -1")

    @property
    def ndof(self) -> int:
        return self.mass.ndof

    @cached_property
    def _engine(self):
        if self.engine is not None:
            return self.engine
        from .engine import Engine, Generators

        if not _is_standard_mass(self.mass):
            raise NotImplementedError("the device kernels implement the P1 criss-cross mass stencil only")
        ny, nx = self.mass.grid_shape
        sx, sy = self.stiff_x, self.stiff_y
        gens = Generators(sx.diag_block.first_col, sx.diag_block.first_row, sx.off_block.first_col,
                          sx.off_block.first_row, sy.diag_block.first_col, sy.diag_block.first_row,
                          sy.off_block.first_col, sy.off_block.first_row, sx.scale, sy.scale, self.mass.scale)
        return Engine(nx, ny, gens, self.kx, self.ky)

    def apply(self, v):
        t, kind = to_device_2d(v, self.ndof)
        eng = self._engine
        if self.half_dt == 0.0:
            return from_device(eng.apply(1, t), kind)
        dt = torch.full((t.shape[0],), 2.0 * self.half_dt, dtype=torch.float64, device=t.device)
        return from_device(eng.apply(0, t, dt, self.sign), kind)

    def dense(self, cap: int = DENSE_CAP) -> np.ndarray:
        out = self.mass.dense(cap)
        if self.half_dt != 0.0:
            out = out + (self.sign * self.half_dt) * (self.kx * self.stiff_x.dense(cap)
                                                      + self.ky * self.stiff_y.dense(cap))
        return out

    def _device_solve(self, rhs, x0, opts: CgOptions):
        b, kind = to_device_2d(rhs, self.ndof)
        counters = torch.zeros(5, dtype=torch.int64, device=b.device)
        x = device_implicit_solve(self._engine, 2.0 * self.half_dt, b, x0, opts, counters)
        return from_device(x, kind), int(counters[1].item())


def device_implicit_solve(engine, dt: float, b: torch.Tensor, x0, opts: CgOptions, counters, group: int = 0):
    """x[b] = [M + dt/2 K]^{-1} b[b] for a batch, CG per system (krylov.py:32-92)."""
    B = b.shape[0]
    dev = b.device
    dts = torch.full((B,), float(dt), dtype=torch.float64, device=dev)
    out = torch.empty_like(b)
    kw = {}
    if x0 is not None:
        xt, _ = to_device_2d(x0, engine.ndof)
        if xt.shape[0] != B:
            xt = xt.expand(B, -1).contiguous()
        kw = dict(x0_mode=2, x0=(xt, -1))
    else:
        kw = dict(x0_mode=0)
    engine.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dts, counters=counters,
                 rel_tol=opts.rel_tol, max_iter=opts.max_iter, explicit=False, f=(b, -1), f_stride=engine.ndof,
                 out=(out, -1), group=group, precond=opts.preconditioner, **kw)
    engine.check_fail()
    return out


def mass_operator(grid: SpatialGrid) -> BttbOperator:
    m1, m2, scale = mass_generators(grid)
    return BttbOperator(scale, m1, m2, axis="x", block_count=grid.my - 1)


def stiffness_operator_x(grid: SpatialGrid, beta: float) -> BttbOperator:
    a1, a2 = stiffness_generators(grid.mx, beta)
    return BttbOperator(stiffness_scale(grid.hx, grid.hy, beta), a1, a2, axis="x", block_count=grid.my - 1)


def stiffness_operator_y(grid: SpatialGrid, gamma: float) -> BttbOperator:
    a1, a2 = stiffness_generators(grid.my, gamma)
    return BttbOperator(stiffness_scale(grid.hy, grid.hx, gamma), a1, a2, axis="y", block_count=grid.mx - 1)


def combined_step_operator(mass, stiff_x, stiff_y, kx, ky, dt, sign, engine=None) -> CombinedStepOperator:
    return CombinedStepOperator(mass, stiff_x, stiff_y, kx, ky, dt / 2.0, sign, engine)


def dense_instantiation(op, cap: int = DENSE_CAP) -> np.ndarray:
    return op.dense(cap)


def permutation_to_column_major(grid: SpatialGrid) -> np.ndarray:
    """x-fastest -> y-fastest index map (test helper, assembly.py:290-301)."""
    return np.arange(grid.ndof).reshape(grid.my - 1, grid.mx - 1).T.ravel()
