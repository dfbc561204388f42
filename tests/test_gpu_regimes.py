"""GPU parity in the step-size regimes the benchmark runs in, against runs of the reference itself.

The round-1 goldens at full spatial size used short horizons (large dt), where the default path's
split-FP16 in-iteration applies never switch on.  These fixtures (tests/golden/make_golden.py) use the
full runs' own fine and coarse step sizes:

* cfg2_split: cfg2 grid/physics, T = 1/8, Nt = 512 (fine dt = 1/4096, level-1 dt = 1/512);
* cfg3_split: cfg3 at 255^2, T = 1/16, Nt = 1024 (fine dt = 1/16384, level-1 1/1024, level-2 1/64) --
  the step sizes of the benchmarked full cfg3 run;
* cfg4_diverge: cfg4 physics (graded mesh, m = 8 multilevel) on 63^2 x 512, where the reference's own
  MGRIT residual grows every cycle; the GPU path must reproduce that trajectory and raise MgritFailure
  carrying the trace and the iterate (reference mgrit.py:317-322, tests/test_mgrit.py:176-182).

Tolerances (north_star): relative L2 <= 1e-10 per time point, identical MGRIT iteration counts and
spatial-solve counts.  Points not stored in full are checked through fixed random projections
("sketches", 8 per point) and norms.
"""

import numpy as np
import pytest

from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.mgrit import MgritFailure, MgritOptions, solve
from paper_1805_06688_b200.stepper import ProblemSpec

pytestmark = pytest.mark.gpu

TOL = 1e-10


def sketch_matrix(ndof, k=8, seed=1234):
    """The projection make_golden.py used (U @ R)."""
    return np.random.default_rng(seed).standard_normal((ndof, k)) / np.sqrt(ndof)


def check_points(U, g, tag, tol=TOL):
    U = np.asarray(U)
    keep = [int(k) for k in g[f"{tag}_keep"]]
    R = g[f"{tag}_U"]
    for k, n in enumerate(keep):
        err = np.linalg.norm(U[n] - R[k]) / max(np.linalg.norm(R[k]), 1e-300)
        assert err <= tol, (n, err)
    ref_norms = g[f"{tag}_norms"]
    norms = np.linalg.norm(U, axis=1)
    assert np.all(np.abs(norms - ref_norms) <= tol * np.maximum(ref_norms, 1e-300))
    # sketch of every point: ||(U_n - R_n) S|| ~ ||U_n - R_n|| sqrt(8/ndof); 5x margin on the chi_8 spread
    S = U @ sketch_matrix(U.shape[1])
    d = np.linalg.norm(S - g[f"{tag}_sketch"], axis=1)
    bound = 5.0 * tol * np.maximum(ref_norms, 1e-300) * np.sqrt(8.0 / U.shape[1])
    bad = np.nonzero(d > bound)[0]
    assert bad.size == 0, (bad[:10], (d / bound)[bad[:10]])


def counters(hier):
    c = np.zeros(5, dtype=np.int64)
    for lv in hier.levels:
        c += lv.disc.counters.cpu().numpy()
    return c


@pytest.mark.parametrize("pre", ["tau", "none"])
@pytest.mark.parametrize("fixture,tag,name,nt,T", [
    ("cfg2_split.npz", "c2p", "cfg2", 512, 0.125),
    ("cfg3_split.npz", "c3p", "cfg3", 1024, 1.0 / 16),
])
def test_benched_regime_matches_reference(golden, fixture, tag, name, nt, T, pre):
    g = golden(fixture)
    case = make_case(name, Nt=nt, T=T)
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol,
                        cg_rel_tol=case.cg_rel_tol, cg_preconditioner=pre)
    hier = []
    U, trace = solve(ProblemSpec(**case.problem_kwargs()), opts, hierarchy_out=hier)
    ref_res = g[f"{tag}_res"]
    assert trace.converged
    assert trace.iterations == len(ref_res) - 1, (trace.residual_norms, ref_res)
    assert np.array_equal(np.array(trace.spatial_solves), g[f"{tag}_solves"])
    check_points(U, g, tag)
    # the residual history: to 1e-6 while it is large; near the halting tolerance the residual is
    # dominated by the inner solves' own 1e-12 tolerance noise (~1e-9 here), which differs between any two
    # correct inner solvers (the reference's plain CG and tau-PCG), so there it agrees to 0.2 halt_tol
    np.testing.assert_allclose(trace.residual_norms, ref_res, rtol=1e-6, atol=0.2 * case.halt_tol)
    if pre == "none":
        # the reference's own (unpreconditioned) CG: the same inner work, which pins the reference-equivalent
        # counts bench.py's CPU extrapolation uses (profiles/<config>_reference_counts.json)
        cg_ref = g[f"{tag}_cgits"]
        assert abs(trace.cg_iterations[-1] - cg_ref[-1]) <= 0.01 * cg_ref[-1] + 2, (trace.cg_iterations, cg_ref)
    if pre == "tau" and name == "cfg2":
        # the regime exists to exercise the split-FP16 in-iteration applies of the default path
        assert counters(hier[0])[4] > 0


def test_cfg4_divergence_matches_reference(golden):
    """cfg4's physics: the reference's MGRIT diverges (re-discretised Crank-Nicolson coarse propagators of
    the stiff fractional operator); the GPU path follows the same trajectory and fails the same way."""
    g = golden("cfg4_diverge.npz")
    case = make_case("cfg4", M=64, Nt=512)
    opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, max_iters=4)
    with pytest.raises(MgritFailure) as info:
        solve(ProblemSpec(**case.problem_kwargs()), opts)
    trace, U = info.value.trace, info.value.solution
    assert not trace.converged
    assert trace.iterations == 4
    np.testing.assert_allclose(trace.residual_norms, g["c4d_res"], rtol=1e-8)
    assert np.array_equal(np.array(trace.spatial_solves), g["c4d_solves"])
    assert np.all(np.diff(trace.residual_norms) > 0)  # grows every cycle, as in the reference
    check_points(U, g, "c4d")


# Accuracy of the default (tau-preconditioned) path on long horizons.  Two correct inner solvers stopped at the
# same relative tolerance 1e-12 land at different points of the tolerance ball, and over thousands of steps
# those differences add up (tools/parity_scan.py, measured on the GPU):
#   cfg2 full (127^2 x 4096): reference's plain CG vs tau-PCG at 1e-12: 4.4e-10; tau-PCG at 1e-13: 4.6e-11;
#     converged answer (inner 1e-14) vs the reference: 2.1e-11;  our plain CG (the reference algorithm): 7e-13.
#   cfg4 physics, full graded grid at 63^2: converged answer vs the reference run: 7.5e-10 (the reference's own
#     1e-12 solves are that far from converged); tau-PCG at any inner tolerance: 7.5e-10; plain CG: 3.4e-13.
# The north_star bar (1e-10 per point) is therefore met by the reference algorithm ('none') everywhere, and by the
# default path wherever the reference run is within ~1e-11 of the converged answer (cfg2 with a 10x tighter inner
# tolerance, cfg3 -- the benchmarked config -- at the reference's own tolerance, test_benched_regime_...).
@pytest.mark.parametrize("pre,tol,bound", [("none", 1e-12, 1e-10), ("tau", 1e-12, 1e-9)])
def test_cfg4_full_graded_grid_matches_reference(golden, pre, tol, bound):
    """cfg4's physics on its full graded time grid (Nt = 8192, t_n = (n/Nt)^2: every fine dt of the BASELINE run,
    levels 8192/1024/128/16/2) at a reduced 63^2 grid, where MGRIT converges: time-dependent propagators at
    every step, parity with the reference's own run."""
    g = golden("cfg4_fullnt.npz")
    case = make_case("cfg4", M=64)
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=tol,
                        cg_preconditioner=pre)
    U, trace = solve(ProblemSpec(**case.problem_kwargs()), opts)
    assert trace.converged
    assert trace.iterations == int(g["c4n_its"])
    assert np.array_equal(np.array(trace.spatial_solves), g["c4n_solves"])
    check_points(U, g, "c4n", tol=bound)
    np.testing.assert_allclose(trace.residual_norms, g["c4n_res"], rtol=1e-6, atol=0.2 * case.halt_tol)


@pytest.mark.parametrize("pre,tol,bound", [("none", 1e-12, 1e-10), ("tau", 1e-13, 1e-10), ("tau", 1e-12, 6e-10)])
def test_cfg2_full_matches_reference(golden, pre, tol, bound):
    """BASELINE configs[1] at full size (127^2 x 4096, multilevel m = 8) against the reference's own full run
    (6,668 s on 4 CPU threads): iteration count, spatial solves, CG totals (reference algorithm), points."""
    g = golden("cfg2_full.npz")
    case = make_case("cfg2")
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=tol,
                        cg_preconditioner=pre)
    U, trace = solve(ProblemSpec(**case.problem_kwargs()), opts)
    assert trace.converged
    assert trace.iterations == int(g["c2f_its"]) == 21
    assert np.array_equal(np.array(trace.spatial_solves), g["c2f_solves"])
    if pre == "none":
        cg_ref = g["c2f_cgits"]
        assert abs(trace.cg_iterations[-1] - cg_ref[-1]) <= 0.01 * cg_ref[-1], (trace.cg_iterations[-1], cg_ref[-1])
    check_points(U, g, "c2f", tol=bound)
    np.testing.assert_allclose(trace.residual_norms, g["c2f_res"], rtol=1e-6, atol=0.2 * case.halt_tol)


def test_cfg5_grid_in_the_full_run_regime_matches_reference(golden):
    """cfg5 grid and physics (1023^2, m = 16) at the full run's step sizes (fine dt = 1/65536, coarse 1/4096;
    two levels at Nt = 32) against the reference's own run: the NP = 1024 large-grid kernel."""
    g = golden("cfg5_split.npz")
    case = make_case("cfg5", Nt=32, T=32.0 / 65536)
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    U, trace = solve(ProblemSpec(**case.problem_kwargs()), opts)
    assert trace.converged
    assert trace.iterations == int(g["c5p_its"])
    assert np.array_equal(np.array(trace.spatial_solves), g["c5p_solves"])
    check_points(U, g, "c5p")
