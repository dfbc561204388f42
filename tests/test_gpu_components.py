"""Component-level parity of the MGRIT building blocks on the GPU path against the oracle's restatement of the same
functions (reference mgrit.py:95-197; the reference's own tests/test_mgrit.py:40-140 check these properties with its
dense 'direct' solver).

Both sides start from the same seeded iterate; each device component (one ``rm_sweep_run`` launch, or the correction
kernel) is compared with the oracle's loop over time points, and the reference tests' structural properties are
asserted on the device result: F-relaxation zeroes the F-point residuals, C-relaxation and the coarse-grid
correction touch C-points only, FCF-relaxation fixes the exact solution, the coarsest solve is forward substitution,
restriction injects the C-point residual.
"""

import numpy as np
import pytest
import torch

from conftest import manufactured
from oracle import riesz_oracle as O
from paper_1805_06688_b200.mesh import SpatialGrid, uniform_temporal
from paper_1805_06688_b200.mgrit import (MgritHierarchy, MgritOptions, c_relax, coarse_correct, exact_solve, f_relax,
                                         fcf_relax, restrict_residual)
from paper_1805_06688_b200.stepper import ProblemSpec, sequential_solve

pytestmark = pytest.mark.gpu
PRECONDS = ["tau", "none"]
TOL = 1e-13      # inner CG (both sides)
CLOSE = 2e-10    # two correct solvers at TOL, a few steps deep


def spec_and_problem(M=8, N=16):
    c = manufactured()
    tm = uniform_temporal(1.0, N)
    spec = ProblemSpec(SpatialGrid(M, M), tm, c["kx"], c["ky"], c["beta"], c["gamma"], c["source"], c["initial"])
    prob = O.Problem(O.Grid(M, M), tm.points, c["kx"], c["ky"], c["beta"], c["gamma"], c["source"], c["initial"])
    return spec, prob


def device_G(level) -> np.ndarray:
    """The level's G as a full [N+1, ndof] array (the fine level may hold it compressed: gscale[n] * gvec)."""
    if level.gscale is None:
        return level.G.cpu().numpy()
    G = np.outer(level.gscale.cpu().numpy(), level.gvec.cpu().numpy())
    G[0] = level.G[0].cpu().numpy()
    return G


def build(pre, N=16, m=4, max_levels=2, seed=0):
    spec, prob = spec_and_problem(N=N)
    hier = MgritHierarchy(spec, MgritOptions(m=m, max_levels=max_levels, cg_rel_tol=TOL, cg_preconditioner=pre))
    levels = O.build_levels(prob, O.Options(m=m, max_levels=max_levels, cg_rel_tol=TOL))
    rng = np.random.default_rng(seed)
    fine, ofine = hier.levels[0], levels[0]
    ofine.U[1:] = rng.random((N, prob.grid.ndof))
    ofine.U[0] = ofine.G[0]
    fine.U.copy_(torch.from_numpy(ofine.U))
    return hier, levels


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-300)))


# ---- hierarchy (mgrit.py:98-134; test_mgrit.py:40-74) -----------------------------------------------------------
def test_automatic_depth_and_caps():
    spec, _ = spec_and_problem(N=16)
    hier = MgritHierarchy(spec, MgritOptions(m=2))
    assert [lv.tmesh.n_intervals for lv in hier.levels] == [16, 8, 4, 2]  # stops at min_coarse
    assert hier.levels[-1].splitting is None
    assert all(lv.splitting is not None for lv in hier.levels[:-1])
    assert MgritHierarchy(spec, MgritOptions(m=2, max_levels=2)).n_levels == 2
    spec12, _ = spec_and_problem(N=12)
    assert [lv.tmesh.n_intervals for lv in MgritHierarchy(spec12, MgritOptions(m=4)).levels] == [12, 3]
    spec2, _ = spec_and_problem(N=2)
    with pytest.warns(UserWarning, match="single level"):
        assert MgritHierarchy(spec2, MgritOptions(m=4)).n_levels == 1


@pytest.mark.parametrize("pre", PRECONDS)
def test_fine_rhs_matches_oracle(pre):
    hier, levels = build(pre, N=8, m=2)
    G = device_G(hier.levels[0])
    assert np.array_equal(G[0], levels[0].G[0])  # the nodal interpolant of psi0
    assert rel(G[1:], levels[0].G[1:]) <= CLOSE


# ---- relaxation (mgrit.py:147-165; test_mgrit.py:77-113) ---------------------------------------------------------
@pytest.mark.parametrize("pre", PRECONDS)
def test_f_relax_matches_oracle_and_zeroes_f_point_residuals(pre):
    hier, levels = build(pre)
    fine, ofine = hier.levels[0], levels[0]
    f_relax(fine)
    hier.check_fail()
    O.f_relax(ofine)
    U = fine.U.cpu().numpy()
    assert rel(U, ofine.U) <= CLOSE
    for n in range(1, 17):
        if n % 4:
            r = ofine.G[n] + ofine.psi(n, U[n - 1]) - U[n]
            assert np.abs(r).max() < 1e-10
        else:
            assert np.array_equal(U[n], ofine.U[n])  # C-points untouched


@pytest.mark.parametrize("pre", PRECONDS)
def test_c_relax_updates_c_points_only(pre):
    hier, levels = build(pre)
    fine, ofine = hier.levels[0], levels[0]
    before = fine.U.cpu().numpy().copy()
    c_relax(fine)
    hier.check_fail()
    O.c_relax(ofine)
    U = fine.U.cpu().numpy()
    for n in range(1, 17):
        if n % 4:
            assert np.array_equal(U[n], before[n])
    assert rel(U[4::4], ofine.U[4::4]) <= CLOSE


@pytest.mark.parametrize("pre", PRECONDS)
def test_fcf_fixes_exact_solution(pre):
    hier, levels = build(pre)
    fine = hier.levels[0]
    exact = O.sequential(levels[0].st.prob, levels[0].st)
    fine.U.copy_(torch.from_numpy(exact))
    fcf_relax(fine)
    hier.check_fail()
    assert np.abs(fine.U.cpu().numpy() - exact).max() < 1e-10


@pytest.mark.parametrize("pre", PRECONDS)
def test_exact_solve_is_forward_substitution(pre):
    hier, levels = build(pre)
    fine, ofine = hier.levels[0], levels[0]
    exact_solve(fine)
    hier.check_fail()
    O.forward_substitution(ofine)
    U = fine.U.cpu().numpy()
    assert rel(U, ofine.U) <= CLOSE
    seq = sequential_solve(fine.disc.spec, fine.disc)
    seq = seq.cpu().numpy() if hasattr(seq, "cpu") else seq
    assert np.abs(U - seq).max() < 1e-9


# ---- restriction and correction (mgrit.py:174-189; test_mgrit.py:115-137) ----------------------------------------
@pytest.mark.parametrize("pre", PRECONDS)
def test_restriction_injects_c_point_residual(pre):
    hier, levels = build(pre)
    restrict_residual(hier, 0)
    hier.check_fail()
    O.restrict(levels[0], levels[1])
    Gc = hier.levels[1].G.cpu().numpy()
    assert np.abs(Gc - levels[1].G).max() <= 1e-10 * max(1.0, np.abs(levels[1].G).max())
    U = hier.levels[0].U.cpu().numpy()
    for k in range(1, 5):
        n = 4 * k
        r = levels[0].G[n] + levels[0].psi(n, U[n - 1]) - U[n]
        assert Gc[k] == pytest.approx(r, abs=1e-10)


@pytest.mark.parametrize("pre", PRECONDS)
def test_coarse_correction_touches_c_points_only(pre):
    hier, _ = build(pre)
    fine, coarse = hier.levels[0], hier.levels[1]
    coarse.U.copy_(torch.from_numpy(np.random.default_rng(1).standard_normal(tuple(coarse.U.shape))))
    before = fine.U.cpu().numpy().copy()
    Uc = coarse.U.cpu().numpy()
    coarse_correct(hier, 0)
    U = fine.U.cpu().numpy()
    for n in range(17):
        if n % 4 == 0:
            assert np.array_equal(U[n], before[n] + Uc[n // 4])
        else:
            assert np.array_equal(U[n], before[n])


# ---- one full two-level cycle against dense algebra (reference tests/test_acceptance.py:293-323, criterion 7) ------
def dense_two_level_propagator(prob: O.Problem, m: int) -> np.ndarray:
    """C-point error propagator of one FCF two-level cycle with re-discretised coarse steps, from dense step matrices:
    J = (I - B^-1 A)(I - A), (A e)_k = e_k - Psi_k e_{k-1} (Psi_k = product of the interval's fine propagators),
    (B e)_k = e_k - Phi_c,k e_{k-1} (one coarse step); k = 0 is the fixed initial value.  Built here from the oracle's
    dense operators -- the reference's error_propagation_oracle (theory.py) is host analysis outside the hot path."""
    ops = O.Operators(prob.grid, prob.kx, prob.ky, prob.beta, prob.gamma)
    n = prob.grid.ndof
    pts = prob.points
    N = pts.size - 1
    Nc = N // m
    phi = lambda dt: np.linalg.solve(ops.step_dense(dt, +1), ops.step_dense(dt, -1))  # noqa: E731
    A = np.eye((Nc + 1) * n)
    B = np.eye((Nc + 1) * n)
    for k in range(1, Nc + 1):
        psi = np.eye(n)
        for j in range((k - 1) * m + 1, k * m + 1):
            psi = phi(pts[j] - pts[j - 1]) @ psi
        A[k * n:(k + 1) * n, (k - 1) * n:k * n] = -psi
        B[k * n:(k + 1) * n, (k - 1) * n:k * n] = -phi(pts[k * m] - pts[(k - 1) * m])
    I = np.eye((Nc + 1) * n)
    return (I - np.linalg.solve(B, A)) @ (I - A)


@pytest.mark.parametrize("pre", PRECONDS)
@pytest.mark.parametrize("mesh_kind", ["uniform", "shishkin"])
@pytest.mark.parametrize("m,N", [(2, 8), (4, 8), (2, 16), (4, 16)])
def test_two_level_cycle_matches_dense_error_propagator(pre, mesh_kind, m, N):
    from paper_1805_06688_b200.mesh import shishkin_temporal

    c = manufactured(0.8, 0.7, 2.0, 0.5)
    tm = uniform_temporal(1.0, N) if mesh_kind == "uniform" else shishkin_temporal(N, 2.0**-4)
    spec = ProblemSpec(SpatialGrid(4, 4), tm, c["kx"], c["ky"], c["beta"], c["gamma"], c["source"], c["initial"])
    prob = O.Problem(O.Grid(4, 4), tm.points, c["kx"], c["ky"], c["beta"], c["gamma"], c["source"], c["initial"])
    hier = MgritHierarchy(spec, MgritOptions(m=m, max_levels=2, cg_rel_tol=TOL, cg_preconditioner=pre))
    fine, coarse = hier.levels
    exact = sequential_solve(spec, fine.disc)
    exact = exact.cpu().numpy() if hasattr(exact, "cpu") else exact
    err = np.random.default_rng(99).standard_normal(exact.shape)
    err[0] = 0.0
    fine.U.copy_(torch.from_numpy(exact + err))
    fcf_relax(fine)
    restrict_residual(hier, 0)
    coarse.U.zero_()
    exact_solve(coarse)
    coarse_correct(hier, 0)
    hier.check_fail()
    got = (fine.U.cpu().numpy() - exact)[::m].ravel()
    predicted = dense_two_level_propagator(prob, m) @ err[::m].ravel()
    assert np.abs(got - predicted).max() <= 1e-9


# ---- property suite across the parameter grid (test_acceptance.py:357-400, criterion 8) ----------------------------
@pytest.mark.parametrize("m", [2, 4, 8, 16])
@pytest.mark.parametrize("pair", [(0.6, 0.7), (0.8, 0.8), (0.95, 0.65)])
def test_fcf_invariance_and_f_residuals_across_parameters(pair, m):
    c = manufactured(*pair, 2.0, 0.5)
    N = 4 * m
    tm = uniform_temporal(1.0, N)
    spec = ProblemSpec(SpatialGrid(4, 4), tm, c["kx"], c["ky"], c["beta"], c["gamma"], c["source"], c["initial"])
    prob = O.Problem(O.Grid(4, 4), tm.points, c["kx"], c["ky"], c["beta"], c["gamma"], c["source"], c["initial"])
    hier = MgritHierarchy(spec, MgritOptions(m=m, max_levels=2, cg_rel_tol=TOL))
    fine = hier.levels[0]
    st = O.Stepper(prob, rel_tol=TOL)
    exact = O.sequential(prob, st)
    fine.U.copy_(torch.from_numpy(exact))
    fcf_relax(fine)
    hier.check_fail()
    assert np.abs(fine.U.cpu().numpy() - exact).max() < 1e-9
    G = device_G(fine)
    U0 = np.random.default_rng(0).random((N + 1, prob.grid.ndof))
    U0[0] = G[0]
    fine.U.copy_(torch.from_numpy(U0))
    fine.ax_valid = False  # U was replaced behind the hierarchy's back
    fcf_relax(fine)
    hier.check_fail()
    U = fine.U.cpu().numpy()
    for n in range(1, N + 1):
        if n % m:
            r = G[n] + st.propagate(tm.points[n] - tm.points[n - 1], U[n - 1]) - U[n]
            assert np.abs(r).max() < 1e-10


@pytest.mark.parametrize("m", [2, 4, 8, 16])
@pytest.mark.parametrize("pair", [(0.6, 0.7), (0.8, 0.8), (0.95, 0.65)])
def test_per_iteration_ratio_respects_two_level_bound(pair, m):
    from paper_1805_06688_b200.mgrit import solve
    from paper_1805_06688_b200.theory import mode_spectrum, two_level_bound

    c = manufactured(*pair, 2.0, 0.5)
    spec = ProblemSpec(SpatialGrid(6, 6), uniform_temporal(1.0, 8 * m), c["kx"], c["ky"], c["beta"], c["gamma"],
                       c["source"], c["initial"])
    bound = two_level_bound(mode_spectrum(spec), spec.tmesh, m).bound
    _, trace = solve(spec, MgritOptions(m=m, max_levels=2, halt_tol=1e-11, cg_rel_tol=TOL))
    norms = trace.residual_norms
    for r_prev, r_next in zip(norms[1:-1], norms[2:]):
        if r_prev < 1e-11:  # measurement floor of the inner solves
            continue
        assert r_next / r_prev <= max(bound, 1e-10) * 1.05 + 1e-12
