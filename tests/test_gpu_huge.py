"""GPU parity at BASELINE config-5 grid size (1023^2 DOF, NP = 1024): the large-grid kernel with 64 CTAs
per chain synchronised through global memory (cooperative launch) instead of a thread-block cluster.

The full config 5 (Nt = 65536, 549 GB of U) needs 8 GPUs; here the spatial operator, one propagation
against the oracle, and a reduced-Nt MGRIT run against sequential time stepping on the same device.
"""

import numpy as np
import pytest

from oracle import riesz_oracle as O
from paper_1805_06688_b200 import assembly
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.krylov import CgOptions
from paper_1805_06688_b200.mesh import SpatialGrid, uniform_temporal
from paper_1805_06688_b200.mgrit import MgritOptions, solve
from paper_1805_06688_b200.stepper import Discretization, ProblemSpec, sequential_solve

pytestmark = pytest.mark.gpu

M, BETA, GAMMA, KX, KY = 1024, 0.7, 0.7, 1.0, 1.0


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_huge_apply_matches_oracle():
    grid = SpatialGrid(M, M)
    ops = O.Operators(O.Grid(M, M), KX, KY, BETA, GAMMA)
    v = np.random.default_rng(0).standard_normal(grid.ndof)
    mass = assembly.mass_operator(grid)
    sx = assembly.stiffness_operator_x(grid, BETA)
    sy = assembly.stiffness_operator_y(grid, GAMMA)
    assert rel(sx.apply(v), ops.sx(v)) <= 1e-13
    assert rel(sy.apply(v), ops.sy(v)) <= 1e-13
    for sign in (1, -1):
        op = assembly.combined_step_operator(mass, sx, sy, KX, KY, 1.0 / 65536, sign)
        assert rel(op.apply(v), ops.step_apply(1.0 / 65536, sign, v)) <= 1e-13


def test_huge_propagate_matches_oracle():
    grid = SpatialGrid(M, M)
    spec = ProblemSpec(grid, uniform_temporal(1.0, 4), KX, KY, BETA, GAMMA, lambda x, y, t: 0 * x,
                       lambda x, y: 0 * x)
    v = np.random.default_rng(1).random(grid.ndof)
    dt = 1.0 / 4096
    st = O.Stepper(O.Problem(O.Grid(M, M), spec.tmesh.points, KX, KY, BETA, GAMMA, spec.source, spec.initial),
                   rel_tol=1e-12)
    want = st.propagate(dt, v)
    for pre in ("tau", "none"):
        disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
        assert rel(disc.propagate(dt, v), want) <= 1e-10


def test_huge_mgrit_matches_sequential():
    """Config 5 structure at Nt = 32 (m = 16, two levels): MGRIT to 1e-8 agrees with sequential time
    stepping to the halting tolerance, and the tau-preconditioned and plain inner solvers agree."""
    case = make_case("cfg5", Nt=32)
    spec = ProblemSpec(**case.problem_kwargs())
    seq = sequential_solve(spec)
    sols = {}
    for pre in ("tau", "none"):
        opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, cg_preconditioner=pre)
        U, tr = solve(spec, opts)
        assert tr.converged and tr.residual_norms[-1] < case.halt_tol
        assert rel(U, seq) <= 1e-7
        sols[pre] = (U, tr)
    assert sols["tau"][1].iterations == sols["none"][1].iterations
    for n in (1, 16, 32):
        assert rel(sols["tau"][0][n], sols["none"][0][n]) <= 1e-10
