"""GPU parity for the large-grid kernels (operand streamed from L2; BASELINE configs 3 and 4 sizes)."""

import numpy as np
import pytest

from oracle import riesz_oracle as O
from paper_1805_06688_b200 import assembly
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.krylov import CgOptions
from paper_1805_06688_b200.mesh import SpatialGrid, uniform_temporal
from paper_1805_06688_b200.mgrit import MgritOptions, solve
from paper_1805_06688_b200.stepper import Discretization, ProblemSpec

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


GRIDS = [(256, 256, 0.75, 0.75, 1.0, 0.5), (200, 150, 0.6, 0.8, 1.0, 2.0), (512, 512, 0.55, 0.9, 1.0, 1.0)]


@pytest.mark.parametrize("mx,my,b,g,kx,ky", GRIDS)
def test_big_apply_matches_oracle(mx, my, b, g, kx, ky):
    grid = SpatialGrid(mx, my)
    ops = O.Operators(O.Grid(mx, my), kx, ky, b, g)
    V = np.random.default_rng(0).standard_normal((2, grid.ndof))
    mass = assembly.mass_operator(grid)
    sx = assembly.stiffness_operator_x(grid, b)
    sy = assembly.stiffness_operator_y(grid, g)
    for k in range(2):
        assert rel(mass.apply(V[k]), ops.mass(V[k])) <= 1e-13
        assert rel(sx.apply(V[k]), ops.sx(V[k])) <= 1e-13
        assert rel(sy.apply(V[k]), ops.sy(V[k])) <= 1e-13
        for sign in (1, -1):
            op = assembly.combined_step_operator(mass, sx, sy, kx, ky, 0.01, sign)
            assert rel(op.apply(V[k]), ops.step_apply(0.01, sign, V[k])) <= 1e-13


@pytest.mark.parametrize("pre", ["none", "tau"])
@pytest.mark.parametrize("mx,my,b,g,kx,ky", GRIDS[:2])
def test_big_propagate_matches_oracle(mx, my, b, g, kx, ky, pre):
    grid = SpatialGrid(mx, my)
    spec = ProblemSpec(grid, uniform_temporal(1.0, 4), kx, ky, b, g, lambda x, y, t: 0 * x, lambda x, y: 0 * x)
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
    st = O.Stepper(O.Problem(O.Grid(mx, my), spec.tmesh.points, kx, ky, b, g, spec.source, spec.initial),
                   rel_tol=1e-12)
    V = np.random.default_rng(1).random((3, grid.ndof))
    for dt in (1.0 / 1024, 1.0 / 16):
        got = disc.propagate(dt, V)
        for k in range(3):
            assert rel(got[k], st.propagate(dt, V[k])) <= 1e-10


@pytest.mark.parametrize("tag,name,nt,pre,fixture", [
    ("c3", "cfg3", 32, "none", "big.npz"),
    ("c3", "cfg3", 32, "tau", "big.npz"),
    ("c4", "cfg4", 16, "none", "big.npz"),
    # at 511^2 the reference's own 1e-12 inner solves are ~2e-10 from the converged answer; the
    # preconditioned path is closer to it, so it is checked against the reference run at 1e-14
    ("c4t", "cfg4", 16, "tau", "big_tight.npz"),
])
def test_big_mgrit_matches_reference(golden, tag, name, nt, pre, fixture):
    try:
        g = golden(fixture)
    except FileNotFoundError:
        pytest.skip(f"{fixture} not generated")
    case = make_case(name, Nt=nt)
    opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, cg_preconditioner=pre)
    U, trace = solve(ProblemSpec(**case.problem_kwargs()), opts)
    ref_res = g[f"{tag}_res"]
    assert trace.iterations == len(ref_res) - 1
    assert np.array_equal(np.array(trace.spatial_solves), g[f"{tag}_solves"])
    assert trace.residual_norms[0] == pytest.approx(float(ref_res[0]), rel=1e-10)
    keep = list(g[f"{tag}_keep"])
    R = g[f"{tag}_U"]
    for k, n in enumerate(keep):
        assert rel(U[n], R[k]) <= 1e-10
    norms = np.linalg.norm(U, axis=1)
    assert np.allclose(norms, g[f"{tag}_norms"], rtol=1e-10, atol=0)


@pytest.mark.parametrize("pre", ["none", "tau"])
def test_big_sequential_and_residual_match_oracle(pre):
    """Large-grid kernel through sequential_solve (rhs F_n + explicit U[n-1], warm start) and
    spacetime_residual (given iterate, x0_mode 2): config-4 structure (graded mesh, f = e^-t g) on 255^2."""
    from paper_1805_06688_b200.stepper import sequential_solve, spacetime_residual

    case = make_case("cfg4", M=256, Nt=6)
    spec = ProblemSpec(**case.problem_kwargs())
    prob = O.Problem(O.Grid(256, 256), spec.tmesh.points, case.kx, case.ky, case.beta, case.gamma, spec.source,
                     spec.initial)
    st = O.Stepper(prob, rel_tol=1e-12)
    R = O.sequential(prob, st)
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
    U = sequential_solve(spec, disc)
    for n in range(R.shape[0]):
        assert rel(U[n], R[n]) <= 1e-10
    Up = R + 1e-3 * np.random.default_rng(5).standard_normal(R.shape)
    norms, tot = spacetime_residual(spec, Up, disc)
    want, wtot = O.spacetime_residual(prob, Up, st)
    assert np.allclose(norms, want, rtol=1e-8, atol=1e-14)
    assert tot == pytest.approx(wtot, rel=1e-8)
