"""Problem description, one-step propagation, sequential stepping (mirrors riesz_mgrit/stepper.py).

    [M + dt/2 (Kx Ax + Ky Ay)] u_n = F_n + [M - dt/2 (Kx Ax + Ky Ay)] u_{n-1}

Every solve runs on the B200 through the chain kernel (one launch per call,
batched over vectors when given a batch).  ``sequential_solve`` and
``spacetime_residual`` are single launches over the whole time grid.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import assembly
from .assembly import device_implicit_solve, from_device, to_device_2d
from .engine import Engine, gauss_tau, require_cuda, to_host
from .krylov import CgOptions
from .loads import HatQuadrature
from .mesh import SpatialGrid, TemporalMesh
from .sources import SeparableP1Source

__all__ = [
    "ProblemSpec",
    "Discretization",
    "initial_vector",
    "load_vector",
    "step",
    "sequential_solve",
    "spacetime_residual",
]


@dataclass(frozen=True)
class ProblemSpec:
    """Riesz diffusion problem, half-orders beta, gamma in (1/2, 1) (stepper.py:37-58)."""

    grid: SpatialGrid
    tmesh: TemporalMesh
    kx: float
    ky: float
    beta: float
    gamma: float
    source: Callable = field(compare=False)
    initial: Callable = field(compare=False)

    def __post_init__(self):
        if self.kx <= 0 or self.ky <= 0:
            raise ValueError("diffusion coefficients must be positive")
        for order in (self.beta, self.gamma):
            if not 0.5 < order < 1.0:
                raise ValueError("fractional half-orders must lie in (1/2, 1)")


class DeviceLoads:
    """F_n on the device for the time points of one level: F_n = fscale[n] * f[n*f_stride]."""

    def __init__(self, f, f_stride, fscale):
        self.f, self.f_stride, self.fscale = f, f_stride, fscale

    def sweep_kwargs(self):
        if self.f is None:
            return {}
        return dict(f=self.f, f_stride=self.f_stride, fscale=self.fscale)


class Discretization:
    """Device operators + counters for one problem (stepper.py:61-146).

    ``solver`` must be 'cg' (the reference's 'direct' dense Cholesky path is a
    <=4096-DOF test device and is out of scope on the GPU).
    """

    def __init__(self, spec: ProblemSpec, cg_opts: CgOptions | None = None, solver: str = "cg",
                 quad_rule: str = "midpoint", quad_refine: int = 1, time_quad_points: int = 2,
                 engine: Engine | None = None):
        if solver not in ("cg", "direct"):
            raise ValueError("solver must be 'cg' or 'direct'")
        if solver == "direct":
            raise NotImplementedError("solver='direct' (dense Cholesky, reference test device) is not provided "
                                      "on the B200 path; use solver='cg'")
        self.spec = spec
        self.cg_opts = cg_opts or CgOptions()
        self.solver = solver
        grid = spec.grid
        self.mass = assembly.mass_operator(grid)
        self.stiff_x = assembly.stiffness_operator_x(grid, spec.beta)
        self.stiff_y = assembly.stiffness_operator_y(grid, spec.gamma)
        self._quad_args = (quad_rule, quad_refine)
        self._quad = None
        self._tq = np.polynomial.legendre.leggauss(time_quad_points)
        self.time_quad_points = time_quad_points
        self.device = require_cuda()
        self.engine = engine or Engine.shared(grid, spec.beta, spec.gamma, spec.kx, spec.ky)
        self.counters = torch.zeros(5, dtype=torch.int64, device=self.device)
        self._combined: dict = {}
        self._mg = None

    @property
    def ndof(self) -> int:
        return self.spec.grid.ndof

    @property
    def spatial_solves(self) -> int:
        return int(self.counters[0].item())

    @property
    def cg_iterations(self) -> int:
        return int(self.counters[1].item())

    def combined(self, dt: float, sign: int) -> assembly.CombinedStepOperator:
        key = (dt, sign)
        if key not in self._combined:
            self._combined[key] = assembly.combined_step_operator(
                self.mass, self.stiff_x, self.stiff_y, self.spec.kx, self.spec.ky, dt, sign, self.engine)
        return self._combined[key]

    def implicit_solve(self, dt: float, rhs, x0=None):
        """Implicit-side solve for one step of size dt (stepper.py:111-122); rhs may be a batch."""
        b, kind = to_device_2d(rhs, self.ndof)
        x = device_implicit_solve(self.engine, dt, b, x0, self.cg_opts, self.counters)
        return from_device(x, kind)

    def propagate(self, dt: float, u_prev):
        """Psi(dt) u_prev: explicit apply + CG warm-started at u_prev (stepper.py:124-127)."""
        v, kind = to_device_2d(u_prev, self.ndof)
        B = v.shape[0]
        dts = torch.full((B,), float(dt), dtype=torch.float64, device=v.device)
        out = torch.empty_like(v)
        self.engine.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dts, counters=self.counters,
                          rel_tol=self.cg_opts.rel_tol, max_iter=self.cg_opts.max_iter, src=v, explicit=True,
                          x0_mode=1, out=(out, -1), precond=self.cg_opts.preconditioner)
        self.engine.check_fail()
        return from_device(out, kind)

    # ------------------------------------------------------------------ loads
    def _separable(self) -> SeparableP1Source | None:
        src = self.spec.source
        if isinstance(src, SeparableP1Source) and src.grid == self.spec.grid and self.time_quad_points == 2:
            return src
        return None

    def mass_times_g(self) -> torch.Tensor:
        if self._mg is None:
            src = self._separable()
            g = torch.from_numpy(np.ascontiguousarray(src.nodal)).to(self.device).reshape(1, -1)
            self._mg = self.engine.apply(1, g)
        return self._mg

    def _quadrature(self) -> HatQuadrature:
        if self._quad is None:
            self._quad = HatQuadrature(self.spec.grid, *self._quad_args)
        return self._quad

    def load_vector(self, t0: float, t1: float) -> np.ndarray:
        """Integral of source * phi_j over [t0, t1] x supp(phi_j) (stepper.py:129-140)."""
        src = self._separable()
        if src is not None:
            if src.kind == "zero":
                return np.zeros(self.ndof)
            tau = gauss_tau(np.array([t0, t1]), src.time_factor)[1]
            return (tau * self.mass_times_g()[0]).cpu().numpy()
        quad = self._quadrature()
        mid, half = (t0 + t1) / 2.0, (t1 - t0) / 2.0
        out = np.zeros(self.ndof)
        for xi, wi in zip(*self._tq):
            fvals = np.asarray(self.spec.source(quad.px, quad.py, mid + half * xi), dtype=float)
            out += (half * wi) * quad.integrate_against_hats(fvals)
        return out

    def device_loads(self, points: np.ndarray) -> DeviceLoads:
        """F_n for n = 1..N of ``points`` in the layout the sweep kernel reads."""
        src = self._separable()
        if src is not None:
            if src.kind == "zero":
                return DeviceLoads(None, 0, None)
            tau = gauss_tau(points, src.time_factor)
            return DeviceLoads(self.mass_times_g(), 0, torch.from_numpy(tau).to(self.device))
        F = np.zeros((points.size, self.ndof))
        for n in range(1, points.size):
            F[n] = self.load_vector(points[n - 1], points[n])
        return DeviceLoads(torch.from_numpy(F).to(self.device), self.ndof, None)

    def rhs_vector(self, n: int) -> np.ndarray:
        """G_n = implicit^{-1} F_n, cold start (stepper.py:142-146)."""
        pts = self.spec.tmesh.points
        return self.implicit_solve(pts[n] - pts[n - 1], self.load_vector(pts[n - 1], pts[n]))


def initial_vector(spec: ProblemSpec) -> np.ndarray:
    """Nodal interpolation of the initial condition (stepper.py:149-152)."""
    x, y = spec.grid.interior_nodes()
    return np.asarray(spec.initial(x, y), dtype=float)


def load_vector(spec: ProblemSpec, n: int, disc: Discretization | None = None) -> np.ndarray:
    if not 1 <= n <= spec.tmesh.n_intervals:
        raise ValueError(f"time index {n} outside 1..{spec.tmesh.n_intervals}")
    disc = disc or Discretization(spec)
    pts = spec.tmesh.points
    return disc.load_vector(pts[n - 1], pts[n])


def step(spec: ProblemSpec, n: int, u_prev, disc: Discretization | None = None):
    """Advance t_{n-1} -> t_n: rhs = F_n + explicit u_prev, x0 = u_prev (stepper.py:163-170)."""
    disc = disc or Discretization(spec)
    pts = spec.tmesh.points
    dt = pts[n] - pts[n - 1]
    rhs = disc.load_vector(pts[n - 1], pts[n]) + disc.combined(dt, -1).apply(u_prev)
    return disc.implicit_solve(dt, rhs, x0=u_prev)


def _dt_tensor(points: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.diff(points)).to(device)


def sequential_solve(spec: ProblemSpec, disc: Discretization | None = None, *, device_result: bool = False):
    """March all time points in one device launch; returns [N+1, ndof] (stepper.py:173-184)."""
    disc = disc or Discretization(spec)
    pts = spec.tmesh.points
    N = spec.tmesh.n_intervals
    U = torch.empty((N + 1, disc.ndof), dtype=torch.float64, device=disc.device)
    U[0] = torch.from_numpy(initial_vector(spec)).to(disc.device)
    loads = disc.device_loads(pts)
    disc.engine.sweep(nchains=1, first=1, cstride=0, clen=N, nmax=N, dt=_dt_tensor(pts, disc.device),
                      counters=disc.counters, rel_tol=disc.cg_opts.rel_tol, max_iter=disc.cg_opts.max_iter,
                      src=U, explicit=True, x0_mode=1, out=U, precond=disc.cg_opts.preconditioner,
                      **loads.sweep_kwargs())
    try:
        disc.engine.check_fail()
    except Exception as exc:
        raise RuntimeError(f"time step {getattr(exc, 'time_index', '?')} failed") from exc
    return U if device_result else to_host(U)


def spacetime_residual(spec: ProblemSpec, U, disc: Discretization | None = None):
    """r_0 = U0_exact - U_0, r_n = implicit^{-1}(F_n + explicit U_{n-1}) - U_n with x0 = U_n.

    Returns (per-point norms [N+1], global norm) (stepper.py:187-205).
    """
    disc = disc or Discretization(spec)
    pts = spec.tmesh.points
    N = spec.tmesh.n_intervals
    Ud, _ = to_device_2d(U, disc.ndof)
    if Ud.shape[0] != N + 1:
        raise ValueError(f"U must have {N + 1} rows")
    sq = torch.zeros(N + 1, dtype=torch.float64, device=disc.device)
    u0 = torch.from_numpy(initial_vector(spec)).to(disc.device)
    disc.engine.diff_sqnorm(u0, Ud[0], sq[0:1])
    loads = disc.device_loads(pts)
    disc.engine.sweep(nchains=N, first=1, cstride=1, clen=1, nmax=N, dt=_dt_tensor(pts, disc.device),
                      counters=disc.counters, rel_tol=disc.cg_opts.rel_tol, max_iter=disc.cg_opts.max_iter,
                      src=Ud, explicit=True, x0_mode=2, x0=Ud, sub=Ud, norms=sq, precond=disc.cg_opts.preconditioner,
                      **loads.sweep_kwargs())
    disc.engine.check_fail()
    norms = np.sqrt(sq.cpu().numpy())
    return norms, float(np.sqrt(np.sum(norms**2)))

