"""Reference edge-case behaviours on the GPU path (reference tests/test_mgrit.py:168-209, tests/test_krylov.py:56-69).

* ``u_init`` = the sequential solution: MGRIT stops before any cycle (test_mgrit.py:168-174);
* the iteration budget raises MgritFailure carrying the trace and the finalized iterate (test_mgrit.py:176-182);
* parareal (F-relaxation, two levels) finishes within N/m + 1 iterations (test_mgrit.py:202-209);
* CG on an indefinite operator (the implicit side with a negative step, through the device sweep) raises
  CgFailure (test_krylov.py:56-60), on the small-grid chain kernel and on the FFT kernel;
* the CG iteration budget raises CgFailure with the budget as its iteration count (test_krylov.py:62-67).
"""

import numpy as np
import pytest

from conftest import manufactured
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.krylov import CgFailure, CgOptions, cg_solve
from paper_1805_06688_b200.mesh import SpatialGrid, uniform_temporal
from paper_1805_06688_b200.mgrit import MgritFailure, MgritOptions, parareal_solve, solve
from paper_1805_06688_b200.stepper import Discretization, ProblemSpec, sequential_solve

pytestmark = pytest.mark.gpu
PRECONDS = ["tau", "none"]


def small_spec(M=8, N=16):
    c = manufactured()
    return ProblemSpec(SpatialGrid(M, M), uniform_temporal(1.0, N), c["kx"], c["ky"], c["beta"], c["gamma"],
                       c["source"], c["initial"])


@pytest.mark.parametrize("pre", PRECONDS)
def test_exact_initial_guess_needs_no_cycle(pre):
    spec = small_spec()
    exact = sequential_solve(spec, Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13, preconditioner=pre)))
    U, trace = solve(spec, MgritOptions(m=4, halt_tol=1e-9, cg_rel_tol=1e-13, cg_preconditioner=pre), u_init=exact)
    assert trace.iterations == 0
    assert trace.converged
    assert np.abs(U - exact).max() < 1e-10


@pytest.mark.parametrize("pre", PRECONDS)
def test_failure_carries_trace_and_iterate(pre):
    spec = small_spec()
    opts = MgritOptions(m=4, max_iters=1, halt_tol=1e-14, cg_rel_tol=1e-12, cg_preconditioner=pre)
    with pytest.raises(MgritFailure) as err:
        solve(spec, opts)
    assert err.value.trace.iterations == 1
    assert not err.value.trace.converged
    assert err.value.solution.shape == (17, spec.grid.ndof)
    assert np.all(np.isfinite(err.value.solution))


@pytest.mark.parametrize("pre", PRECONDS)
def test_parareal_terminates_within_coarse_interval_count(pre):
    spec = small_spec(N=16)
    _, trace = parareal_solve(spec, MgritOptions(m=4, halt_tol=1e-9, cg_rel_tol=1e-12, cg_preconditioner=pre))
    assert trace.converged
    assert trace.iterations <= 16 // 4 + 1


@pytest.mark.parametrize("pre", PRECONDS)
@pytest.mark.parametrize("grid", ["small", "fft"])
def test_indefinite_operator_breaks_down(pre, grid):
    """M + (dt/2) K with a large negative dt has negative eigenvalues: p'Ap <= 0 (or a non-finite
    preconditioned residual) -> CgFailure, as the reference's CG raises on an indefinite operator."""
    spec = small_spec(M=16, N=4) if grid == "small" else ProblemSpec(**make_case("cfg3", Nt=4).problem_kwargs())
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
    b = np.random.default_rng(0).standard_normal(disc.ndof)
    with pytest.raises(CgFailure):
        cg_solve(disc.combined(-50.0, +1), b, opts=CgOptions(rel_tol=1e-12, preconditioner=pre))


@pytest.mark.parametrize("pre", PRECONDS)
def test_iteration_budget(pre):
    spec = small_spec(M=16, N=4)
    disc = Discretization(spec)
    b = np.random.default_rng(1).standard_normal(disc.ndof)
    with pytest.raises(CgFailure) as err:
        cg_solve(disc.combined(0.5, +1), b, opts=CgOptions(rel_tol=1e-14, max_iter=2, preconditioner=pre))
    assert err.value.iterations == 2


# ---- scalability proxy and spatial-solve overhead model (reference tests/test_acceptance.py:405-447, criterion 9; the
# reference runs them with its dense 'direct' solver, here the CG paths of the device kernels) ----------------------
def _proxy_spec(M, N):
    c = manufactured(0.6, 0.7, 2.0, 0.5)
    return ProblemSpec(SpatialGrid(M, M), uniform_temporal(1.0, N), c["kx"], c["ky"], c["beta"], c["gamma"],
                       c["source"], c["initial"])


@pytest.mark.parametrize("pre", PRECONDS)
def test_iteration_count_stable_in_N(pre):
    counts = []
    for N in (256, 1024, 4096):
        _, trace = solve(_proxy_spec(16, N), MgritOptions(m=4, halt_tol=1e-9, cg_rel_tol=1e-12, cg_preconditioner=pre))
        assert trace.converged
        counts.append(trace.iterations)
    assert max(counts) - min(counts) <= 2, counts


@pytest.mark.parametrize("pre", PRECONDS)
def test_spatial_solve_overhead_model(pre):
    """One multilevel cycle costs about (2m/(m-1) + 1) solves per coarse interval summed over the hierarchy, linear in N;
    sequential stepping costs exactly N solves."""
    m = 4
    per_cycle = {}
    for N in (512, 1024):
        opts = MgritOptions(m=m, halt_tol=1e-9, cg_rel_tol=1e-12, skip_first_down=False, cg_preconditioner=pre)
        _, trace = solve(_proxy_spec(8, N), opts)
        per_cycle[N] = float(np.mean(np.diff(trace.spatial_solves)[1:]))
        coarse_sum, n_l = 0, N
        while n_l % m == 0 and n_l // m >= 2:
            coarse_sum += n_l // m
            n_l //= m
        model = (2 * m / (m - 1) + 1) * coarse_sum
        assert 0.25 <= model / per_cycle[N] <= 4.0, (per_cycle[N], model)
    assert per_cycle[1024] / per_cycle[512] == pytest.approx(2.0, rel=0.25)
    spec = _proxy_spec(8, 512)
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
    sequential_solve(spec, disc)
    assert disc.spatial_solves == 512
