"""Canonical seeded inputs for the BASELINE.json configurations.

BASELINE.json fixes the physics of five configurations but not the seeds or
the draw order, so this module pins them ("canonical recipe").  The same
recipe feeds the reference/oracle runs and the GPU runs, so both see
bit-identical inputs.  All data are synthetic (no dataset is involved).

Data RNG is ``np.random.default_rng(0)`` drawn in the order listed:

* cfg1: psi0 = x(1-x)y(1-y)(1 + 0.01 N(0,1)), then g ~ U(-1,1), s(t) = 1
* cfg2: psi0 = sin(pi x) sin(pi y) + 1e-3 N(0,1), then g ~ U(-1,1), s(t) = t
* cfg3: c ~ N(0,1)^{4x4}, psi0 = sum c_kl sin(k pi x) sin(l pi y), f = 0
* cfg4: psi0 as cfg2 but from default_rng(1); g from default_rng(0); s(t) = exp(-t);
        graded mesh t_n = (n/Nt)^2
* cfg5: psi0 = sin(pi x) sin(pi y), g ~ U(-1,1), s(t) = 1
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import SpatialGrid, TemporalMesh, graded_temporal, uniform_temporal
from .sources import NodalInitial, SeparableP1Source

__all__ = ["CaseSpec", "make_case", "CONFIGS"]


@dataclass
class CaseSpec:
    name: str
    grid: SpatialGrid
    tmesh: TemporalMesh
    kx: float
    ky: float
    beta: float
    gamma: float
    psi0: np.ndarray = field(repr=False)
    g: np.ndarray = field(repr=False)
    kind: str
    m: int
    max_levels: int | None
    halt_tol: float = 1e-8
    cg_rel_tol: float = 1e-12

    @property
    def source(self) -> SeparableP1Source:
        return SeparableP1Source(self.grid, self.g, self.kind)

    @property
    def initial(self) -> NodalInitial:
        return NodalInitial(self.grid, self.psi0)

    def problem_kwargs(self):
        """Keyword arguments for a reference-style ProblemSpec."""
        return dict(grid=self.grid, tmesh=self.tmesh, kx=self.kx, ky=self.ky,
                    beta=self.beta, gamma=self.gamma, source=self.source, initial=self.initial)


# name -> (M cells per direction, Nt, beta, gamma, kx, ky, m, max_levels)
CONFIGS = {
    "cfg1": (32, 256, 0.7, 0.7, 1.0, 1.0, 4, 2),
    "cfg2": (128, 4096, 0.6, 0.8, 1.0, 2.0, 8, None),
    "cfg3": (256, 16384, 0.75, 0.75, 1.0, 0.5, 16, None),
    "cfg4": (512, 8192, 0.55, 0.9, 1.0, 1.0, 8, None),
    "cfg5": (1024, 65536, 0.7, 0.7, 1.0, 1.0, 16, None),
}


def make_case(name: str, M: int | None = None, Nt: int | None = None,
              max_levels: int | None | str = "default", T: float = 1.0) -> CaseSpec:
    """Build a configuration; ``M``/``Nt`` override the sizes (reduced parity cases); ``T`` the final time
    (BASELINE: T = 1; bench.py's weak scaling extends the horizon at a fixed step, T = Nt / Nt_config)."""
    M0, Nt0, beta, gamma, kx, ky, m, lv = CONFIGS[name]
    M = M0 if M is None else M
    Nt = Nt0 if Nt is None else Nt
    if max_levels != "default":
        lv = max_levels
    grid = SpatialGrid(M, M)
    x, y = grid.interior_nodes()
    n = grid.ndof
    sxy = np.sin(np.pi * x) * np.sin(np.pi * y)
    tmesh = uniform_temporal(T, Nt)
    if name == "cfg1":
        rng = np.random.default_rng(0)
        psi0 = x * (1 - x) * y * (1 - y) * (1.0 + 0.01 * rng.standard_normal(n))
        g = rng.uniform(-1.0, 1.0, n)
        kind = "one"
    elif name == "cfg2":
        rng = np.random.default_rng(0)
        psi0 = sxy + 1e-3 * rng.standard_normal(n)
        g = rng.uniform(-1.0, 1.0, n)
        kind = "t"
    elif name == "cfg3":
        rng = np.random.default_rng(0)
        c = rng.standard_normal((4, 4))
        psi0 = np.zeros(n)
        for k in range(1, 5):
            for l in range(1, 5):
                psi0 += c[k - 1, l - 1] * np.sin(k * np.pi * x) * np.sin(l * np.pi * y)
        g = np.zeros(n)
        kind = "zero"
    elif name == "cfg4":
        psi0 = sxy + 1e-3 * np.random.default_rng(1).standard_normal(n)
        g = np.random.default_rng(0).uniform(-1.0, 1.0, n)
        kind = "exp_neg_t"
        tmesh = graded_temporal(T, Nt, 2.0)
    elif name == "cfg5":
        rng = np.random.default_rng(0)
        psi0 = sxy.copy()
        g = rng.uniform(-1.0, 1.0, n)
        kind = "one"
    else:
        raise KeyError(name)
    return CaseSpec(name, grid, tmesh, kx, ky, beta, gamma, psi0, g, kind, m, lv)
