"""CPU oracle: a numpy restatement of the reference hot path (riesz_mgrit 0.1.0).

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module.  It may be used by ``tests/``, ``__graft_entry__.smoke()`` (as the
checker) and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs (as the
timed CPU implementation of the path).  It is never the thing measured for
the GPU arm and never a fallback.

Parity pinning: every function below is checked against golden vectors that
were produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.

Reference file:line citations are relative to ``/root/reference/pkg/src/riesz_mgrit``.
The arithmetic is deliberately the reference's: dense Toeplitz blocks applied
with numpy ``@`` (OpenBLAS DGEMM), unpreconditioned CG with the reference's
stopping rule, serial Python sweeps.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable

import numpy as np
from numpy.polynomial.legendre import leggauss
from scipy.linalg import toeplitz
from scipy.sparse import csr_matrix

# ----------------------------------------------------------------------------
# Grids (mesh.py:20-58, 61-92, 125-161)
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class Grid:
    """mx*my cells on the unit square (mesh.py:20-58); unknowns x-fastest."""

    mx: int
    my: int

    @property
    def hx(self):
        return 1.0 / self.mx

    @property
    def hy(self):
        return 1.0 / self.my

    @property
    def nx(self):
        return self.mx - 1

    @property
    def ny(self):
        return self.my - 1

    @property
    def ndof(self):
        return self.nx * self.ny

    def nodes(self):
        """Interior node coordinates, x fastest (mesh.py:47-52)."""
        xs = self.hx * np.arange(1, self.mx)
        ys = self.hy * np.arange(1, self.my)
        X, Y = np.meshgrid(xs, ys)
        return X.ravel(), Y.ravel()


def uniform_points(T: float, N: int) -> np.ndarray:
    """mesh.py:125-131."""
    return np.linspace(0.0, T, N + 1)


def level_points(points: np.ndarray, m: int, max_levels, min_coarse: int = 2):
    """Temporal hierarchy by injection (mgrit.py:107-116, mesh.py:157-161)."""
    N = points.size - 1
    if max_levels is None:
        max_levels = int(math.floor(math.log(N, m))) + 1 if N >= m else 1
    out = [np.asarray(points, dtype=float)]
    while len(out) < max_levels:
        n = out[-1].size - 1
        if n % m or n // m < min_coarse:
            break
        out.append(out[-1][::m].copy())
    return out


# ----------------------------------------------------------------------------
# Generators (assembly.py:172-251) and BTTB apply (assembly.py:100-115)
# ----------------------------------------------------------------------------


def mass_blocks(n: int):
    """Dense (M1, M2) Toeplitz blocks of order n (assembly.py:172-187)."""
    c1 = np.zeros(n)
    c1[0] = 6.0
    if n > 1:
        c1[1] = 1.0
    c2 = np.zeros(n)
    r2 = np.zeros(n)
    c2[0] = r2[0] = 1.0
    if n > 1:
        r2[1] = 1.0
    return toeplitz(c1, c1), toeplitz(c2, r2)


def stiffness_gens(M: int, rho: float):
    """(first col/row of A1, first col of A2, first row of A2) (assembly.py:190-251)."""
    if not 0.5 < rho < 1.0:
        raise ValueError("fractional half-order must lie in (1/2, 1)")
    if M < 2:
        raise ValueError("need at least 2 intervals")
    n = M - 1
    q3 = 3.0 - 2.0 * rho
    q4 = 4.0 - 2.0 * rho
    a = np.zeros(n)
    a[0] = 2.0 ** (6.0 - 2.0 * rho) + 16.0 * rho - 40.0
    if n > 1:
        a[1] = 2.0 * 3.0**q4 + (2.0 * rho - 6.0) * 2.0 ** (5.0 - 2.0 * rho) - 16.0 * rho + 34.0
    if n > 2:
        j = np.arange(2.0, n)
        a[2:] = (4.0 * q4 * (2.0 * j**q3 - (j - 1.0) ** q3 - (j + 1.0) ** q3)
                 - 2.0 * (j - 2.0) ** q4 + 4.0 * (j - 1.0) ** q4
                 - 4.0 * (j + 1.0) ** q4 + 2.0 * (j + 2.0) ** q4)
    d = 4.0 - 2.0**q4 * rho
    row = np.zeros(n)
    col = np.zeros(n)
    row[0] = col[0] = d
    if n > 1:
        row[1] = d
    if n > 2:
        j = np.arange(2.0, n)
        row[2:] = (q4 * ((j - 2.0) ** q3 - (j - 1.0) ** q3 - j**q3 + (j + 1.0) ** q3)
                   + 2.0 * (j - 2.0) ** q4 - 6.0 * (j - 1.0) ** q4
                   + 6.0 * j**q4 - 2.0 * (j + 1.0) ** q4)
    if n > 1:
        j = np.arange(1.0, n)
        col[1:] = (q4 * ((j - 1.0) ** q3 - j**q3 - (j + 1.0) ** q3 + (j + 2.0) ** q3)
                   + 2.0 * (j - 1.0) ** q4 - 6.0 * j**q4
                   + 6.0 * (j + 1.0) ** q4 - 2.0 * (j + 2.0) ** q4)
    return a, col, row


def stiffness_scale(h_along: float, h_across: float, rho: float) -> float:
    """Prefactor of assembly.py:259-274."""
    return h_along ** (1.0 - 2.0 * rho) * h_across / (
        2.0 * math.cos(rho * math.pi) * math.gamma(5.0 - 2.0 * rho))


@dataclass
class Bttb:
    """scale * (I (x) T1 + S (x) T2 + S^T (x) T2^T) in x- or y-block form."""

    scale: float
    T1: np.ndarray
    T2: np.ndarray
    axis: str
    shape: tuple  # (ny, nx)

    def __call__(self, v: np.ndarray) -> np.ndarray:
        # assembly.py:100-115: three DGEMMs per call on the 2-D view
        V = np.asarray(v, dtype=float).reshape(self.shape)
        if self.axis == "x":
            W = V @ self.T1.T
            W[:-1] += V[1:] @ self.T2.T
            W[1:] += V[:-1] @ self.T2
        else:
            W = self.T1 @ V
            W[:, :-1] += self.T2 @ V[:, 1:]
            W[:, 1:] += self.T2.T @ V[:, :-1]
        return self.scale * W.ravel()

    def dense(self) -> np.ndarray:
        ny, nx = self.shape
        if self.axis == "x":
            up = np.eye(ny, k=1)
            full = np.kron(np.eye(ny), self.T1) + np.kron(up, self.T2) + np.kron(up.T, self.T2.T)
        else:
            up = np.eye(nx, k=1)
            full = np.kron(self.T1, np.eye(nx)) + np.kron(self.T2, up) + np.kron(self.T2.T, up.T)
        return self.scale * full


@dataclass
class Operators:
    """Mass and directional stiffness of one spatial grid (assembly.py:254-274)."""

    grid: Grid
    kx: float
    ky: float
    beta: float
    gamma: float
    mass: Bttb = field(init=False)
    sx: Bttb = field(init=False)
    sy: Bttb = field(init=False)

    def __post_init__(self):
        g = self.grid
        shape = (g.ny, g.nx)
        M1, M2 = mass_blocks(g.nx)
        self.mass = Bttb(g.hx * g.hy / 12.0, M1, M2, "x", shape)
        a, c, r = stiffness_gens(g.mx, self.beta)
        self.sx = Bttb(stiffness_scale(g.hx, g.hy, self.beta), toeplitz(a, a), toeplitz(c, r), "x", shape)
        a, c, r = stiffness_gens(g.my, self.gamma)
        self.sy = Bttb(stiffness_scale(g.hy, g.hx, self.gamma), toeplitz(a, a), toeplitz(c, r), "y", shape)

    def step_apply(self, dt: float, sign: int, v: np.ndarray) -> np.ndarray:
        """(M + sign*dt/2*(kx Ax + ky Ay)) v  (assembly.py:155-161, :277-286)."""
        hd = dt / 2.0
        out = self.mass(v)
        if hd != 0.0:
            out = out + (sign * hd) * (self.kx * self.sx(v) + self.ky * self.sy(v))
        return out

    def step_dense(self, dt: float, sign: int) -> np.ndarray:
        hd = dt / 2.0
        return self.mass.dense() + (sign * hd) * (self.kx * self.sx.dense() + self.ky * self.sy.dense())


# ----------------------------------------------------------------------------
# CG (krylov.py:32-92)
# ----------------------------------------------------------------------------


class OracleCgFailure(RuntimeError):
    def __init__(self, msg, residual_norm, iterations):
        super().__init__(msg)
        self.residual_norm = residual_norm
        self.iterations = iterations


def cg(apply, b, x0=None, rel_tol=1e-9, max_iter=None):
    """Unpreconditioned CG with the reference stopping rule; returns (x, its)."""
    b = np.asarray(b, dtype=float)
    n = b.size
    kmax = 10 * n if max_iter is None else max_iter
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=float)
    bnorm = np.linalg.norm(b)
    tol = rel_tol * bnorm if bnorm > 0 else rel_tol
    r = b - apply(x)
    rn = np.linalg.norm(r)
    if rn <= tol:
        return x, 0
    p = r.copy()
    rho = rn**2
    k = 0
    while k < kmax:
        k += 1
        q = apply(p)
        pq = p @ q
        if not np.isfinite(pq) or pq <= 0:
            raise OracleCgFailure(f"breakdown at {k}", rn, k)
        a = rho / pq
        x += a * p
        r -= a * q
        rho_new = r @ r
        rn = np.sqrt(rho_new)
        if not np.isfinite(rn):
            raise OracleCgFailure(f"non-finite residual at {k}", rn, k)
        if rn <= tol:
            # acceptance test on the true residual (krylov.py:71-83)
            tr = np.linalg.norm(b - apply(x))
            if tr <= max(tol, 10 * rn):
                return x, k
            r = b - apply(x)
            rho_new = r @ r
            rn = np.sqrt(rho_new)
            if rn <= tol:
                return x, k
            p = r.copy()
            rho = rho_new
            continue
        p = r + (rho_new / rho) * p
        rho = rho_new
    raise OracleCgFailure("iteration budget exhausted", rn, kmax)


# ----------------------------------------------------------------------------
# Source quadrature (quadrature.py:23-131, stepper.py:129-140)
# ----------------------------------------------------------------------------


def _tri_rule_midpoint_refined(refine: int):
    """Edge-midpoint rule in barycentric form, subdivided `refine` times (quadrature.py:23-67)."""
    base = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])
    tris = [np.eye(3)]
    for _ in range(refine):
        nxt = []
        for t in tris:
            a, b, c = t
            ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
            nxt += [np.array([a, ab, ca]), np.array([ab, b, bc]), np.array([ca, bc, c]), np.array([ab, bc, ca])]
        tris = nxt
    pts = np.vstack([base @ t for t in tris])
    w = np.full(pts.shape[0], 1.0 / pts.shape[0])
    return pts, w


class LoadQuadrature:
    """Hat-function load vectors on the criss-cross triangulation (quadrature.py:70-131)."""

    def __init__(self, grid: Grid, refine: int = 1, time_points: int = 2):
        self.grid = grid
        bary, w = _tri_rule_midpoint_refined(refine)
        mx, my = grid.mx, grid.my
        ci, cj = np.meshgrid(np.arange(mx), np.arange(my))
        ci, cj = ci.ravel(), cj.ravel()
        node = lambda i, j: j * (mx + 1) + i  # noqa: E731
        tri = np.vstack([
            np.stack([node(ci, cj), node(ci + 1, cj), node(ci + 1, cj + 1)], axis=1),
            np.stack([node(ci, cj), node(ci + 1, cj + 1), node(ci, cj + 1)], axis=1),
        ])
        gx = np.tile(grid.hx * np.arange(mx + 1), my + 1)
        gy = np.repeat(grid.hy * np.arange(my + 1), mx + 1)
        self.px = (gx[tri] @ bary.T).ravel()
        self.py = (gy[tri] @ bary.T).ravel()
        dof = -np.ones((mx + 1) * (my + 1), dtype=np.int64)
        jj, ii = np.meshgrid(np.arange(1, my), np.arange(1, mx), indexing="ij")
        dof[(jj * (mx + 1) + ii).ravel()] = np.arange(grid.ndof)
        area = grid.hx * grid.hy / 2.0
        q = bary.shape[0]
        pid = np.arange(tri.shape[0] * q).reshape(tri.shape[0], q)
        rows, cols, vals = [], [], []
        for v in range(3):
            d = dof[tri[:, v]]
            keep = d >= 0
            for k in range(q):
                rows.append(d[keep])
                cols.append(pid[keep, k])
                vals.append(np.full(keep.sum(), area * w[k] * bary[k, v]))
        self.W = csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                            shape=(grid.ndof, tri.shape[0] * q))
        self.tnodes, self.tweights = leggauss(time_points)

    def load(self, source: Callable, t0: float, t1: float) -> np.ndarray:
        """2-point Gauss in time x spatial quadrature (stepper.py:129-140)."""
        mid, half = (t0 + t1) / 2.0, (t1 - t0) / 2.0
        out = np.zeros(self.grid.ndof)
        for xi, wi in zip(self.tnodes, self.tweights):
            f = np.asarray(source(self.px, self.py, mid + half * xi), dtype=float)
            out += (half * wi) * (self.W @ f)
        return out


# ----------------------------------------------------------------------------
# Stepper (stepper.py:61-205)
# ----------------------------------------------------------------------------


@dataclass
class Problem:
    grid: Grid
    points: np.ndarray
    kx: float
    ky: float
    beta: float
    gamma: float
    source: Callable
    initial: Callable


class Stepper:
    """Per-level operators + solve counters (stepper.py:61-146)."""

    def __init__(self, prob: Problem, rel_tol: float = 1e-9):
        self.prob = prob
        self.ops = Operators(prob.grid, prob.kx, prob.ky, prob.beta, prob.gamma)
        self.rel_tol = rel_tol
        self.quad = None
        self.solves = 0
        self.cg_its = 0

    def solve(self, dt, b, x0=None):
        """Implicit-side solve (stepper.py:111-122)."""
        self.solves += 1
        x, its = cg(lambda v: self.ops.step_apply(dt, +1, v), b, x0=x0, rel_tol=self.rel_tol)
        self.cg_its += its
        return x

    def propagate(self, dt, v):
        """Psi v: explicit apply then CG warm-started at v (stepper.py:124-127)."""
        return self.solve(dt, self.ops.step_apply(dt, -1, v), x0=v)

    def load(self, n):
        if self.quad is None:
            self.quad = LoadQuadrature(self.prob.grid)
        p = self.prob.points
        return self.quad.load(self.prob.source, p[n - 1], p[n])

    def g_vector(self, n):
        """G_n = implicit^{-1} F_n, cold start (stepper.py:142-146)."""
        p = self.prob.points
        return self.solve(p[n] - p[n - 1], self.load(n))


def initial_nodal(prob: Problem) -> np.ndarray:
    x, y = prob.grid.nodes()
    return np.asarray(prob.initial(x, y), dtype=float)


def sequential(prob: Problem, st: Stepper | None = None) -> np.ndarray:
    """stepper.py:163-184: rhs = F_n + explicit U[n-1], x0 = U[n-1]."""
    st = st or Stepper(prob)
    p = prob.points
    N = p.size - 1
    U = np.empty((N + 1, prob.grid.ndof))
    U[0] = initial_nodal(prob)
    for n in range(1, N + 1):
        dt = p[n] - p[n - 1]
        U[n] = st.solve(dt, st.load(n) + st.ops.step_apply(dt, -1, U[n - 1]), x0=U[n - 1])
    return U


def spacetime_residual(prob: Problem, U: np.ndarray, st: Stepper | None = None):
    """stepper.py:187-205: per-point norms and global norm, x0 = U[n]."""
    st = st or Stepper(prob)
    p = prob.points
    N = p.size - 1
    norms = np.empty(N + 1)
    norms[0] = np.linalg.norm(initial_nodal(prob) - U[0])
    for n in range(1, N + 1):
        dt = p[n] - p[n - 1]
        rhs = st.load(n) + st.ops.step_apply(dt, -1, U[n - 1])
        norms[n] = np.linalg.norm(st.solve(dt, rhs, x0=U[n]) - U[n])
    return norms, float(np.sqrt(np.sum(norms**2)))


# ----------------------------------------------------------------------------
# MGRIT (mgrit.py:79-337)
# ----------------------------------------------------------------------------


@dataclass
class Level:
    points: np.ndarray
    st: Stepper
    m: int | None  # None on the coarsest level
    G: np.ndarray
    U: np.ndarray

    @property
    def N(self):
        return self.points.size - 1

    def psi(self, n, v):
        """Psi_n with dt = t_n - t_{n-1} of this level (mgrit.py:89-92)."""
        return self.st.propagate(self.points[n] - self.points[n - 1], v)


@dataclass
class Options:
    m: int
    max_levels: int | None = None
    min_coarse: int = 2
    halt_tol: float = 1e-9
    max_iters: int = 100
    relaxation: str = "fcf"
    skip_first_down: bool = True
    rng_seed: int = 0
    cg_rel_tol: float = 1e-9


class OracleMgritFailure(RuntimeError):
    def __init__(self, msg, trace, solution):
        super().__init__(msg)
        self.trace = trace
        self.solution = solution


def build_levels(prob: Problem, opts: Options):
    """mgrit.py:98-134 (fine G computed with cold-start solves)."""
    pts = level_points(prob.points, opts.m, opts.max_levels, opts.min_coarse)
    levels = []
    for i, p in enumerate(pts):
        st = Stepper(replace(prob, points=p), rel_tol=opts.cg_rel_tol)
        N = p.size - 1
        levels.append(Level(p, st, None if i == len(pts) - 1 else opts.m,
                            np.zeros((N + 1, prob.grid.ndof)), np.zeros((N + 1, prob.grid.ndof))))
    fine = levels[0]
    fine.G[0] = initial_nodal(prob)
    for n in range(1, fine.N + 1):
        fine.G[n] = fine.st.g_vector(n)
    return levels


def f_relax(lv: Level, U=None):
    """mgrit.py:147-156."""
    U = lv.U if U is None else U
    for base in range(0, lv.N, lv.m):
        v = U[base]
        for n in range(base + 1, min(base + lv.m, lv.N + 1)):
            v = lv.psi(n, v) + lv.G[n]
            U[n] = v


def c_relax(lv: Level, U=None):
    """mgrit.py:159-165."""
    U = lv.U if U is None else U
    U[0] = lv.G[0]
    for n in range(lv.m, lv.N + 1, lv.m):
        U[n] = lv.psi(n, U[n - 1]) + lv.G[n]


def restrict(fine: Level, coarse: Level):
    """mgrit.py:174-182."""
    m = fine.m
    coarse.G[0] = fine.G[0] - fine.U[0]
    for k in range(1, coarse.N + 1):
        n = k * m
        coarse.G[k] = fine.G[n] + fine.psi(n, fine.U[n - 1]) - fine.U[n]


def correct(fine: Level, coarse: Level):
    """mgrit.py:185-189."""
    fine.U[::fine.m] += coarse.U


def forward_substitution(lv: Level):
    """mgrit.py:192-197."""
    lv.U[0] = lv.G[0]
    for n in range(1, lv.N + 1):
        lv.U[n] = lv.psi(n, lv.U[n - 1]) + lv.G[n]


def v_cycle(levels, opts: Options, l=0, skip=False):
    """mgrit.py:200-221."""
    lv = levels[l]
    if lv.m is None:
        forward_substitution(lv)
        return
    if not skip:
        f_relax(lv)
        if opts.relaxation == "fcf":
            c_relax(lv)
            f_relax(lv)
    restrict(lv, levels[l + 1])
    levels[l + 1].U[:] = 0.0
    v_cycle(levels, opts, l + 1, skip)
    correct(lv, levels[l + 1])
    if l > 0:
        f_relax(lv)


def residual_norm(levels):
    """mgrit.py:253-273: F-relax a copy, sum initial + C-point residuals."""
    lv = levels[0]
    V = lv.U.copy()
    sq = float(np.sum((lv.G[0] - V[0]) ** 2))
    if lv.m is None:
        idx = range(1, lv.N + 1)
    else:
        f_relax(lv, V)
        idx = range(lv.m, lv.N + 1, lv.m)
    for n in idx:
        r = lv.G[n] + lv.psi(n, V[n - 1]) - V[n]
        sq += float(r @ r)
    return math.sqrt(sq), V


@dataclass
class Trace:
    residual_norms: list = field(default_factory=list)
    spatial_solves: list = field(default_factory=list)
    cg_iterations: list = field(default_factory=list)
    converged: bool = False

    @property
    def iterations(self):
        return len(self.residual_norms) - 1


def mgrit_solve(prob: Problem, opts: Options, u_init=None):
    """mgrit.py:276-322; returns (finalized U, trace)."""
    levels = build_levels(prob, opts)
    fine = levels[0]
    if u_init is not None:
        fine.U[:] = np.asarray(u_init, dtype=float)
    else:
        fine.U[1:] = np.random.default_rng(opts.rng_seed).random((fine.N, prob.grid.ndof))
    fine.U[0] = fine.G[0]
    tr = Trace()

    def rec(norm):
        tr.residual_norms.append(norm)
        tr.spatial_solves.append(sum(lv.st.solves for lv in levels))
        tr.cg_iterations.append(sum(lv.st.cg_its for lv in levels))

    norm, V = residual_norm(levels)
    rec(norm)
    if norm < opts.halt_tol:
        tr.converged = True
        return V, tr
    for it in range(1, opts.max_iters + 1):
        v_cycle(levels, opts, 0, skip=opts.skip_first_down and it == 1)
        norm, V = residual_norm(levels)
        rec(norm)
        if norm < opts.halt_tol:
            tr.converged = True
            return V, tr
    raise OracleMgritFailure("no convergence", tr, V)


def parareal(prob: Problem, opts: Options):
    """mgrit.py:325-327."""
    return mgrit_solve(prob, replace(opts, relaxation="f", max_levels=2))


# ----------------------------------------------------------------------------
# numpy PCG64 stream (the reference's initial guess, mgrit.py:291-292)
# ----------------------------------------------------------------------------

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1


def pcg64_state(seed: int):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    return int(st["state"]), int(st["inc"])


def pcg64_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """Pure-python PCG64 XSL-RR doubles (draws start..start+count-1)."""
    s, inc = pcg64_state(seed)
    s = pcg64_advance(s, inc, start)
    out = np.empty(count)
    for i in range(count):
        s = (s * PCG_MULT + inc) & MASK128
        x = ((s >> 64) ^ s) & MASK64
        rot = s >> 122
        x = ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64
        out[i] = (x >> 11) * (1.0 / 9007199254740992.0)
    return out


def pcg64_advance(s: int, inc: int, delta: int) -> int:
    """LCG jump-ahead by delta steps (Brown 1994)."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = PCG_MULT, inc
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        delta >>= 1
    return (acc_mult * s + acc_plus) & MASK128
