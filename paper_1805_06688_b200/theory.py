"""A-priori two-level MGRIT convergence bound (mirrors riesz_mgrit/theory.py:50-142).

Host-side analysis, not on the hot path: every one-step propagator of the Crank-Nicolson-type scheme
(stepper.py:3-6) shares the eigenvectors of the generalised problem (Kx Ax + Ky Ay) x = sigma M x and
acts on mode sigma as the scalar (2 - dt sigma) / (2 + dt sigma) (theory.py:68-71).  The two-level error
and residual reduction factor is bounded by the maximum over modes of

    (lam+)^m |(lam+)^m - mu-| (1 - (mu*)^(Nc-1)) / (1 - mu*)                       (theory.py:88-134)

with lam+ = max_j |lambda_j| over the fine step widths, mu- the signed minimum and mu* the maximum
modulus of the coarse factors.  For the reference's dense eigensolve the spatial order is capped at
assembly.DENSE_CAP (theory.py:50-65); the spectra here come from the same dense operators on the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import assembly
from .mesh import TemporalMesh, coarsen

__all__ = ["ModeSpectrum", "BoundReport", "mode_spectrum", "step_factors", "two_level_bound",
           "residual_ratio_bound"]


@dataclass(frozen=True)
class ModeSpectrum:
    """Sorted generalised eigenvalues sigma > 0 of (Kx Ax + Ky Ay, M) (theory.py:37-47)."""

    sigmas: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "sigmas", np.asarray(self.sigmas, dtype=float))

    @property
    def n_modes(self) -> int:
        return self.sigmas.size


def mode_spectrum(spec, cap: int = assembly.DENSE_CAP) -> ModeSpectrum:
    """Dense symmetric-definite eigensolve of the spatial pencil (theory.py:50-65); raises ValueError above
    ``cap`` unknowns and RuntimeError on a non-positive eigenvalue (a broken assembly)."""
    import scipy.linalg

    grid = spec.grid
    if grid.ndof > cap:
        raise ValueError(f"spatial dimension {grid.ndof} exceeds dense cap {cap}")
    mass = assembly.mass_operator(grid).dense(cap)
    stiff = spec.kx * assembly.stiffness_operator_x(grid, spec.beta).dense(cap)
    stiff = stiff + spec.ky * assembly.stiffness_operator_y(grid, spec.gamma).dense(cap)
    sym = lambda a: 0.5 * (a + a.T)  # noqa: E731  (exact symmetry for the definite solver)
    sigmas = scipy.linalg.eigh(sym(stiff), sym(mass), eigvals_only=True)
    if sigmas[0] <= 0:
        raise RuntimeError(f"non-positive eigenvalue {sigmas[0]:.3e}: operator assembly is broken")
    return ModeSpectrum(np.sort(sigmas))


def step_factors(sigma, dt):
    """Propagator eigenvalue (2 - dt sigma) / (2 + dt sigma), in (-1, 1) (theory.py:68-71)."""
    x = np.multiply(dt, sigma)
    return (2.0 - x) / (2.0 + x)


@dataclass
class BoundReport:
    """The bound and its per-mode ingredients (theory.py:74-85)."""

    bound: float
    argmax_mode: int
    lam_dagger: np.ndarray
    mu_ddagger: np.ndarray
    mu_star: np.ndarray
    per_mode: np.ndarray
    m: int
    n_coarse: int


def _geometric_sums(mu_star: np.ndarray, n_coarse: int) -> np.ndarray:
    """sum_{i < Nc-1} (mu*)^i per mode; the closed form away from mu* = 1, the explicit sum next to it."""
    if n_coarse < 2:
        return np.zeros_like(mu_star)  # one coarse interval: the coarse solve is exact
    out = np.empty_like(mu_star)
    near = np.abs(1.0 - mu_star) < 1e-8
    far = ~near
    out[far] = (1.0 - mu_star[far] ** (n_coarse - 1)) / (1.0 - mu_star[far])
    if near.any():
        p = np.arange(n_coarse - 1)
        out[near] = (mu_star[near][:, None] ** p[None, :]).sum(axis=1)
    return out


def two_level_bound(spectrum: ModeSpectrum, fine_mesh: TemporalMesh, m: int, chunk: int = 256) -> BoundReport:
    """Two-level bound on a uniform or graded fine mesh with coarsening factor m (theory.py:88-134)."""
    if fine_mesh.n_intervals % m:
        raise ValueError(f"factor {m} does not divide N={fine_mesh.n_intervals}")
    coarse = coarsen(fine_mesh, m)
    wf = np.unique(fine_mesh.widths)
    wc = np.unique(coarse.widths)
    sig = spectrum.sigmas
    lam_dagger = np.empty_like(sig)
    mu_ddagger = np.empty_like(sig)
    mu_star = np.empty_like(sig)
    for lo in range(0, sig.size, chunk):  # modes in chunks: (widths x modes) stays small on graded meshes
        s = sig[lo:lo + chunk][None, :]
        lam = step_factors(s, wf[:, None])
        mu = step_factors(s, wc[:, None])
        lam_dagger[lo:lo + s.shape[1]] = np.abs(lam).max(axis=0)
        mu_ddagger[lo:lo + s.shape[1]] = mu.min(axis=0)
        mu_star[lo:lo + s.shape[1]] = np.abs(mu).max(axis=0)
    per_mode = lam_dagger ** m * np.abs(lam_dagger ** m - mu_ddagger) * _geometric_sums(mu_star,
                                                                                         coarse.n_intervals)
    k = int(np.argmax(per_mode))
    return BoundReport(float(per_mode[k]), k, lam_dagger, mu_ddagger, mu_star, per_mode, m, coarse.n_intervals)


def residual_ratio_bound(spectrum: ModeSpectrum, fine_mesh: TemporalMesh, m: int) -> float:
    """Bound on successive fine-grid residual ratios: the same expression (theory.py:137-141)."""
    return two_level_bound(spectrum, fine_mesh, m).bound
