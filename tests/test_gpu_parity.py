"""GPU parity: the CUDA path (through the C ABI) against golden vectors produced by
running the reference itself (tests/golden/make_golden.py).

Tolerances (FP64, stated per check):
  * operator applies: relative L2 <= 1e-13 (reference pins 1e-12 abs vs dense,
    tests/test_assembly.py:116-124);
  * single solves at rel_tol 1e-12..1e-13: relative L2 <= 1e-10;
  * MGRIT / sequential solutions: relative L2 <= 1e-10 PER TIME POINT and the
    SAME iteration count (BASELINE.json north_star), identical solve counts.
"""

import numpy as np
import pytest
import torch

from conftest import manufactured

pytestmark = pytest.mark.gpu

from paper_1805_06688_b200 import assembly  # noqa: E402
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.krylov import CgOptions, cg_solve  # noqa: E402
from paper_1805_06688_b200.mesh import SpatialGrid, TemporalMesh, uniform_temporal  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, parareal_solve, solve  # noqa: E402
from paper_1805_06688_b200.stepper import (  # noqa: E402
    Discretization,
    ProblemSpec,
    sequential_solve,
    spacetime_residual,
)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def per_point_rel(U, R):
    U = np.asarray(U)
    R = np.asarray(R)
    num = np.linalg.norm(U - R, axis=1)
    den = np.maximum(np.linalg.norm(R, axis=1), 1e-300)
    return num / den


def man_spec(M, N, **kw):
    c = manufactured(**kw)
    return ProblemSpec(SpatialGrid(M, M), uniform_temporal(1.0, N), c["kx"], c["ky"], c["beta"], c["gamma"],
                       c["source"], c["initial"])


# ----------------------------------------------------------------------------- operators
@pytest.mark.parametrize("case", range(5))
def test_operator_apply_matches_reference(golden, case):
    g = golden("operators.npz")
    mx, my, b, gm, kx, ky = g[f"c{case}_params"]
    grid = SpatialGrid(int(mx), int(my))
    mass = assembly.mass_operator(grid)
    sx = assembly.stiffness_operator_x(grid, b)
    sy = assembly.stiffness_operator_y(grid, gm)
    V = g[f"c{case}_v"]
    assert rel(mass.apply(V), g[f"c{case}_mass"]) <= 1e-13
    assert rel(sx.apply(V), g[f"c{case}_sx"]) <= 1e-13
    assert rel(sy.apply(V), g[f"c{case}_sy"]) <= 1e-13
    for sign, tag in ((1, "imp"), (-1, "exp")):
        for k, dt in enumerate(g[f"c{case}_dts"]):
            op = assembly.combined_step_operator(mass, sx, sy, kx, ky, dt, sign)
            assert rel(op.apply(V[k]), g[f"c{case}_{tag}"][k]) <= 1e-13, (tag, dt)


def test_apply_accepts_device_batches(golden):
    g = golden("operators.npz")
    mx, my, b, gm, kx, ky = g["c3_params"]
    grid = SpatialGrid(int(mx), int(my))
    sx = assembly.stiffness_operator_x(grid, b)
    V = torch.from_numpy(g["c3_v"]).cuda()
    out = sx.apply(V)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert rel(out.cpu().numpy(), g["c3_sx"]) <= 1e-13


# ----------------------------------------------------------------------------- CG
PRECONDS = ["none", "tau", "tau16", "tau64"]


@pytest.mark.parametrize("pre", PRECONDS)
@pytest.mark.parametrize("k", range(4))
def test_cg_matches_reference(golden, k, pre):
    g = golden("cg.npz")
    M, dt, warm, tol = g[f"k{k}_params"]
    spec = man_spec(int(M), 4, beta=0.6, gamma=0.7)
    disc = Discretization(spec)
    op = disc.combined(dt, +1)
    x0 = g[f"k{k}_x0"] if warm else None
    x, its = cg_solve(op, g[f"k{k}_b"], x0=x0, opts=CgOptions(rel_tol=tol, preconditioner=pre))
    assert rel(x, g[f"k{k}_x"]) <= 1e-9
    if pre == "none":
        assert abs(its - int(g[f"k{k}_its"])) <= 1
    else:
        assert its <= int(g[f"k{k}_its"])
    # the reference's residual criterion on the returned iterate
    r = g[f"k{k}_b"] - op.apply(x)
    assert np.linalg.norm(r) <= 10 * tol * np.linalg.norm(g[f"k{k}_b"])


def test_cg_warm_start_at_solution_takes_zero_iterations(golden):
    g = golden("cg.npz")
    spec = man_spec(16, 4, beta=0.6, gamma=0.7)
    disc = Discretization(spec)
    op = disc.combined(0.01, +1)
    b = g["k0_b"]
    x, _ = cg_solve(op, b, opts=CgOptions(rel_tol=1e-13))
    x2, its = cg_solve(op, b, x0=x, opts=CgOptions(rel_tol=1e-9))
    assert its == 0
    assert np.array_equal(x2, x)


def test_cg_zero_rhs():
    disc = Discretization(man_spec(8, 4))
    x, its = cg_solve(disc.combined(0.1, +1), np.zeros(disc.ndof))
    assert its == 0 and not np.any(x)


def test_cg_budget_failure_raises():
    from paper_1805_06688_b200.krylov import CgFailure

    disc = Discretization(man_spec(16, 4))
    b = np.random.default_rng(1).standard_normal(disc.ndof)
    with pytest.raises(CgFailure) as err:
        cg_solve(disc.combined(1.0, +1), b, opts=CgOptions(rel_tol=1e-14, max_iter=2))
    assert err.value.iterations == 2


# cg_solve with an arbitrary operator (krylov.py:44; the reference's tests/test_krylov.py cases): same algorithm,
# vectors and reductions on the device (rm_vec_dot / rm_vec_axpby), the operator called once per iteration
class _SpdOperator:
    def __init__(self, dense):
        self.dense = dense

    def apply(self, v):
        return self.dense @ v


def _random_spd(n, rng, cond=100.0):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return Q @ np.diag(np.geomspace(1.0, cond, n)) @ Q.T


def test_generic_cg_matches_direct_solve_and_oracle():
    rng = np.random.default_rng(12345)
    A = _random_spd(40, rng)
    b = rng.standard_normal(40)
    x, iters = cg_solve(_SpdOperator(A), b, opts=CgOptions(rel_tol=1e-12))
    assert x == pytest.approx(np.linalg.solve(A, b), abs=1e-8)
    from oracle import riesz_oracle as O

    xo, io = O.cg(lambda v: A @ v, b, rel_tol=1e-12)
    assert iters == io and np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)


def test_generic_cg_accepts_plain_callable_and_device_operator():
    rng = np.random.default_rng(3)
    A = _random_spd(10, rng)
    b = rng.standard_normal(10)
    x, _ = cg_solve(lambda v: A @ v, b, opts=CgOptions(rel_tol=1e-12))
    assert A @ x == pytest.approx(b, abs=1e-9)
    At = torch.from_numpy(A).cuda()

    class Dev:
        accepts_device = True

        def apply(self, v):
            return At @ v

    xd, _ = cg_solve(Dev(), torch.from_numpy(b).cuda(), opts=CgOptions(rel_tol=1e-12))
    assert xd.is_cuda and xd.cpu().numpy() == pytest.approx(x, abs=1e-9)


def test_generic_cg_warm_start_zero_rhs_and_tolerance():
    rng = np.random.default_rng(5)
    A = _random_spd(20, rng)
    b = rng.standard_normal(20)
    x_exact = np.linalg.solve(A, b)
    x, iters = cg_solve(_SpdOperator(A), b, x0=x_exact)
    assert iters == 0 and x == pytest.approx(x_exact)
    x, iters = cg_solve(_SpdOperator(A), np.zeros(20))
    assert iters == 0 and x == pytest.approx(np.zeros(20))
    A = _random_spd(30, rng, cond=1e4)
    b = rng.standard_normal(30)
    x, _ = cg_solve(_SpdOperator(A), b, opts=CgOptions(rel_tol=1e-10))
    assert np.linalg.norm(b - A @ x) <= 1e-10 * np.linalg.norm(b) * 10


def test_generic_cg_failures():
    from paper_1805_06688_b200.krylov import CgFailure

    with pytest.raises(CgFailure):
        cg_solve(_SpdOperator(np.diag([1.0, -1.0, 2.0, -2.0])), np.ones(4))
    rng = np.random.default_rng(7)
    A = _random_spd(50, rng, cond=1e8)
    with pytest.raises(CgFailure) as err:
        cg_solve(_SpdOperator(A), rng.standard_normal(50), opts=CgOptions(rel_tol=1e-14, max_iter=2))
    assert err.value.iterations == 2


def test_generic_cg_runs_the_package_operators():
    """The explicit-side operator (and any BttbOperator) goes through the generic route with its device apply."""
    disc = Discretization(man_spec(8, 4))
    op = disc.combined(1e-3, -1)  # M - s K at a small step: SPD
    b = np.random.default_rng(2).standard_normal(disc.ndof)
    x, iters = cg_solve(op, b, opts=CgOptions(rel_tol=1e-12))
    assert iters > 0 and np.linalg.norm(op.apply(x) - b) <= 1e-11 * np.linalg.norm(b)


# ----------------------------------------------------------------------------- stepper
def test_stepper_matches_reference(golden):
    g = golden("stepper.npz")
    spec = man_spec(4, 8)
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13))
    pts = spec.tmesh.points
    loads = np.stack([disc.load_vector(pts[n - 1], pts[n]) for n in range(1, 9)])
    assert rel(loads, g["loads"]) <= 1e-14
    gv = np.stack([disc.rhs_vector(n) for n in range(1, 9)])
    assert rel(gv, g["gvecs"]) <= 1e-10
    assert rel(disc.propagate(0.125, g["prop_v"]), g["prop_out"]) <= 1e-10
    seq = sequential_solve(spec, Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13)))
    assert per_point_rel(seq, g["seq"]).max() <= 1e-10
    U = g["seq"].copy()
    U[3] += 1e-3
    norms, tot = spacetime_residual(spec, U, Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13)))
    assert np.allclose(norms, g["stres_norms"], rtol=1e-8, atol=1e-12)
    assert tot == pytest.approx(float(g["stres_total"]), rel=1e-8)


def test_sequential_16_matches_reference(golden):
    g = golden("stepper.npz")
    spec = man_spec(16, 32)
    U = sequential_solve(spec, Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12)))
    assert per_point_rel(U, g["seq16"]).max() <= 1e-10


# ----------------------------------------------------------------------------- MGRIT
SMALL_RUNS = {
    "two": dict(m=4, max_levels=2),
    "multi": dict(m=4),
    "noskip": dict(m=4, skip_first_down=False),
    "frelax": dict(m=2, relaxation="f"),
    "seed3": dict(m=8, rng_seed=3),
}


def check_run(U, trace, g, tag, pre="none"):
    ref_res = g[f"{tag}_res"]
    assert trace.iterations == len(ref_res) - 1, (trace.residual_norms, ref_res)
    assert trace.converged
    assert np.array_equal(np.array(trace.spatial_solves), g[f"{tag}_solves"])
    # the initial residual depends only on the (bit-identical) initial guess and G
    assert trace.residual_norms[0] == pytest.approx(float(ref_res[0]), rel=1e-10)
    cg_ref = g[f"{tag}_cgits"]
    if pre == "none":  # the reference's unpreconditioned CG: same work
        assert abs(trace.cg_iterations[-1] - cg_ref[-1]) <= 0.01 * cg_ref[-1] + 2
    else:  # preconditioned inner solves: fewer iterations, same solutions
        assert trace.cg_iterations[-1] < cg_ref[-1]
    R = g[f"{tag}_U"]
    if R.shape[0] != np.asarray(U).shape[0]:
        U = np.asarray(U)[:: (np.asarray(U).shape[0] - 1) // (R.shape[0] - 1)]
    assert per_point_rel(U, R).max() <= 1e-10


@pytest.mark.parametrize("pre", PRECONDS)
@pytest.mark.parametrize("tag", list(SMALL_RUNS))
def test_small_mgrit_matches_reference(golden, tag, pre):
    g = golden("mgrit_small.npz")
    spec = man_spec(8, 64)
    opts = MgritOptions(halt_tol=1e-10, cg_rel_tol=1e-12, cg_preconditioner=pre, **SMALL_RUNS[tag])
    U, trace = solve(spec, opts)
    check_run(U, trace, g, tag, pre)


@pytest.mark.parametrize("pre", PRECONDS)
def test_small_parareal_matches_reference(golden, pre):
    g = golden("mgrit_small.npz")
    U, trace = parareal_solve(man_spec(8, 64), MgritOptions(m=8, halt_tol=1e-10, cg_rel_tol=1e-12,
                                                            cg_preconditioner=pre))
    check_run(U, trace, g, "parareal", pre)


def case_spec(case):
    return ProblemSpec(**case.problem_kwargs())


@pytest.mark.parametrize("pre", PRECONDS)
@pytest.mark.parametrize("tag,levels", [("two", 2), ("multi", None)])
def test_cfg1_matches_reference(golden, tag, levels, pre):
    g = golden("cfg1.npz")
    case = make_case("cfg1")
    assert np.array_equal(case.psi0, g["psi0"]) and np.array_equal(case.g, g["g"])
    opts = MgritOptions(m=case.m, max_levels=levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol,
                        cg_preconditioner=pre)
    U, trace = solve(case_spec(case), opts)
    check_run(U, trace, g, tag, pre)
    # MGRIT vs sequential time stepping (tests/test_mgrit.py:137-144 uses 1e-8)
    assert np.abs(U - g["seq_U"]).max() <= 1e-8


@pytest.mark.parametrize("pre", PRECONDS)
def test_cfg1_sequential_matches_reference(golden, pre):
    g = golden("cfg1.npz")
    case = make_case("cfg1")
    spec = case_spec(case)
    U = sequential_solve(spec, Discretization(spec, cg_opts=CgOptions(rel_tol=case.cg_rel_tol, preconditioner=pre)))
    assert per_point_rel(U, g["seq_U"]).max() <= 1e-10


@pytest.mark.parametrize("tag,name,kw", [
    ("g_two", "cfg4", dict(M=16, Nt=64, levels=2)),
    ("g_multi", "cfg4", dict(M=16, Nt=64, levels=None)),
    ("c2", "cfg2", dict(M=None, Nt=16, levels=None)),
    ("c2s", "cfg2", dict(M=32, Nt=512, levels=None)),
])
@pytest.mark.parametrize("pre", PRECONDS)
def test_reduced_configs_match_reference(golden, tag, name, kw, pre):
    g = golden("reduced.npz")
    case = make_case(name, M=kw["M"], Nt=kw["Nt"])
    opts = MgritOptions(m=case.m, max_levels=kw["levels"], halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol,
                        cg_preconditioner=pre)
    U, trace = solve(case_spec(case), opts)
    check_run(U, trace, g, tag, pre)


# ----------------------------------------------------------------------------- RNG, determinism
def test_device_pcg64_is_numpy_bit_exact(golden):
    from paper_1805_06688_b200.engine import Engine

    g = golden("pcg64.npz")
    eng = Engine.for_problem(SpatialGrid(4, 4), 0.7, 0.7, 1.0, 1.0)
    out = torch.empty((8, 16129), dtype=torch.float64, device="cuda")
    eng.pcg64_fill(0, out)
    flat = out.cpu().numpy().ravel()
    assert np.array_equal(flat[g["offsets"]], g["values"])
    assert np.array_equal(flat[:16], g["first"])
    assert np.array_equal(flat, np.random.default_rng(0).random((8, 16129)).ravel())


@pytest.mark.parametrize("pre", PRECONDS)
@pytest.mark.parametrize("M", [32, 64, 128])
def test_results_independent_of_cluster_size(M, pre):
    """Chains processed by 1, 2, 4, 8 or 16 CTAs give bitwise identical results."""
    from paper_1805_06688_b200 import _native
    from paper_1805_06688_b200.engine import Engine

    case = make_case("cfg2", M=M, Nt=8)
    eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
    n = case.grid.ndof
    V = torch.from_numpy(np.random.default_rng(5).random((6, n))).cuda()
    dt = torch.full((6,), 1.0 / 64, dtype=torch.float64, device="cuda")
    outs = []
    np_ = 16
    while np_ < M - 1:
        np_ *= 2
    for G in (1, 2, 4, 8, 16):
        lib = _native.lib()
        if not _supported(np_, G):
            continue
        out = torch.zeros_like(V)
        cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
        norms = torch.zeros(7, dtype=torch.float64, device="cuda")
        eng.sweep(nchains=6, first=1, cstride=1, clen=1, nmax=6, dt=dt, counters=cnt, rel_tol=1e-12, src=V,
                  x0_mode=1, out=(out, -1), norms=(norms, -1), group=G, precond=pre)
        eng.check_fail()
        outs.append((G, out.cpu().numpy(), norms.cpu().numpy(), cnt.cpu().numpy()))
        del lib
    assert len(outs) >= 2
    for G, o, nr, c in outs[1:]:
        assert np.array_equal(o, outs[0][1]), G
        assert np.array_equal(nr, outs[0][2]), G
        assert np.array_equal(c, outs[0][3]), G


def _supported(np_, G):
    table = {16: (1,), 32: (1, 2), 64: (1, 2, 4), 128: (2, 4, 8, 16)}
    return G in table[np_]


def test_solve_is_deterministic():
    case = make_case("cfg1", Nt=32)
    opts = MgritOptions(m=4, halt_tol=1e-8, cg_rel_tol=1e-12)
    U1, t1 = solve(case_spec(case), opts)
    U2, t2 = solve(case_spec(case), opts)
    assert t1.residual_norms == t2.residual_norms
    assert np.array_equal(U1, U2)


def test_graded_mesh_uses_per_step_dt():
    case = make_case("cfg4", M=8, Nt=16)
    assert not case.tmesh.is_uniform()
    spec = case_spec(case)
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12))
    U = sequential_solve(spec, disc)
    # one propagation at step n with its own dt reproduces the sequential update
    n = 7
    w = spec.tmesh.widths[n - 1]
    pts = spec.tmesh.points
    rhs = disc.load_vector(pts[n - 1], pts[n]) + disc.combined(w, -1).apply(U[n - 1])
    x = disc.implicit_solve(w, rhs, x0=U[n - 1])
    assert rel(x, U[n]) <= 1e-12


@pytest.mark.parametrize("dt", [1.0 / 4096, 1.0 / 64, 1.0 / 8])
def test_tau_preconditioner_cuts_iterations(dt):
    """127^2 cfg2 operator: PCG reaches the reference tolerance in far fewer iterations."""
    case = make_case("cfg2", Nt=8)
    spec = case_spec(case)
    v = np.random.default_rng(4).random((4, case.grid.ndof))
    out = {}
    for pre in PRECONDS:
        disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
        out[pre] = (disc.propagate(dt, v), disc.cg_iterations)
    assert per_point_rel(out["tau"][0], out["none"][0]).max() <= 1e-10
    assert out["tau"][1] * 2 <= out["none"][1] or dt < 1e-3
    assert out["tau"][1] < out["none"][1]
    # FP16 DST stages (FP32 accumulation) leave the PCG iteration count essentially unchanged
    assert abs(out["tau16"][1] - out["tau64"][1]) <= max(1, 0.05 * out["tau64"][1])
    # split-FP16 applies inside the iteration: same FP64 stopping test, at most a restart's worth more
    assert out["tau"][1] <= 1.5 * out["tau64"][1] + 4
    for pre in ("tau", "tau16"):
        assert per_point_rel(out[pre][0], out["tau64"][0]).max() <= 1e-10


@pytest.mark.parametrize("M,cfg", [(6, "cfg1"), (16, "cfg1"), (32, "cfg1"), (64, "cfg2"), (128, "cfg2")])
def test_preconditioner_probe_matches_numpy(M, cfg):
    """z = P(s)^-1 b from the device (rm_sweep x0_mode 3) against precond.py's tau diagonals and dense DST
    matrices: FP64 DST stages to rounding, FP16 stages (FP32 accumulation) to FP16 accuracy."""
    from paper_1805_06688_b200.engine import Engine
    from paper_1805_06688_b200.precond import dst_matrix, tau_diagonals

    case = make_case(cfg, M=M, Nt=8)
    g = case.grid
    eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
    dm, dk = tau_diagonals(g, case.beta, case.gamma, case.kx, case.ky)
    Sx, Sy = dst_matrix(g.nx), dst_matrix(g.ny)
    rng = np.random.default_rng(M)
    V = rng.standard_normal((3, g.ndof)) * np.array([[1.0], [1e-9], [1e6]])
    dts = np.array([1.0 / 4096, 1.0 / 64, 0.5])
    ref = np.stack([(Sy @ ((Sy @ v.reshape(g.ny, g.nx) @ Sx) / (dm + 0.5 * dt * dk)) @ Sx).ravel()
                    for v, dt in zip(V, dts)])
    Vd, dtd = torch.from_numpy(V).cuda(), torch.from_numpy(dts).cuda()
    z64 = eng.precond_apply(Vd, dtd, "tau64").cpu().numpy()
    z16 = eng.precond_apply(Vd, dtd, "tau").cpu().numpy()
    for k in range(3):
        assert rel(z64[k], ref[k]) <= 1e-12, (k, rel(z64[k], ref[k]))
        assert rel(z16[k], ref[k]) <= 5e-3, (k, rel(z16[k], ref[k]))


@pytest.mark.parametrize("M,cfg", [(64, "cfg2"), (128, "cfg2")])
def test_split_fp16_apply_probe(M, cfg):
    """The in-iteration split-FP16 apply (rm_sweep x0_mode 4) against the FP64 apply on random, smooth and
    oscillating vectors: a few ulp of FP32 relative to sum |terms|."""
    from paper_1805_06688_b200.engine import Engine

    case = make_case(cfg, M=M, Nt=8)
    g = case.grid
    eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
    rng = np.random.default_rng(M)
    x, y = np.meshgrid(np.arange(1, g.nx + 1) / (g.nx + 1), np.arange(1, g.ny + 1) / (g.ny + 1))
    V = np.stack([rng.standard_normal(g.ndof), (np.sin(np.pi * x) * np.sin(np.pi * y)).ravel(),
                  rng.standard_normal(g.ndof) * 1e-20, ((-1.0) ** np.arange(g.ndof)) * 3e5])
    dts = np.array([1.0 / 4096, 1.0 / 64, 0.5, 1.0 / 512])
    Vd, dtd = torch.from_numpy(V).cuda(), torch.from_numpy(dts).cuda()
    lp = eng.lp_apply_probe(Vd, dtd).cpu().numpy()
    ref = np.stack([eng.apply(0, Vd[k:k + 1], dtd[k:k + 1], +1).cpu().numpy()[0] for k in range(4)])
    for k in range(4):
        print(k, rel(lp[k], ref[k]))
        assert rel(lp[k], ref[k]) <= 1e-5, (k, rel(lp[k], ref[k]))


@pytest.mark.parametrize("cfg,M,Nt", [("cfg2", 32, 256), ("cfg2", 128, 64), ("cfg1", None, 64)])
def test_apply_reuse_matches_applied_path(cfg, M, Nt, monkeypatch):
    """The apply-free chain right-hand sides and stored-A x second guesses (rm_sweep d_hg / d_ax / d_gax) give the
    same MGRIT trajectory as applying the operator: identical iteration and solve counts, per-point solutions
    within the solve tolerance."""
    case = make_case(cfg, M=M, Nt=Nt)
    spec = case_spec(case)
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    out = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("RM_NO_APPLY_REUSE", flag)
        out[flag] = solve(spec, opts)
    (U0, t0), (U1, t1) = out["0"], out["1"]
    assert t0.iterations == t1.iterations
    assert t0.spatial_solves == t1.spatial_solves
    assert per_point_rel(U0, U1).max() <= 1e-10
