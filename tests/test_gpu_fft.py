"""The FFT chain kernel (csrc/rm_fft.cu; 255^2 grids, BASELINE config 3) against the CPU oracle.

Its operator is evaluated through 512-point FFTs (circulant embedding of the Toeplitz blocks) and its tau
preconditioner's DST-I through odd-extended FFTs, all in FP64: the probes below pin both against the
oracle's dense operator (reference assembly.py:100-115, 155-161) and the numpy DST preconditioner
(precond.py), and propagations against the oracle's CG (krylov.py:32-92).
"""

import numpy as np
import pytest
import torch

from oracle import riesz_oracle as O
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.engine import Engine
from paper_1805_06688_b200.precond import dst_matrix, tau_diagonals
from paper_1805_06688_b200.krylov import CgOptions
from paper_1805_06688_b200.stepper import Discretization, ProblemSpec

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def vectors(g, rng):
    x, y = np.meshgrid(np.arange(1, g.nx + 1) / (g.nx + 1), np.arange(1, g.ny + 1) / (g.ny + 1))
    return np.stack([rng.standard_normal(g.ndof), (np.sin(np.pi * x) * np.sin(np.pi * y)).ravel(),
                     rng.random(g.ndof), ((-1.0) ** np.arange(g.ndof)) * 3e5])


@pytest.mark.parametrize("name", ["cfg3"])
def test_fft_apply_matches_oracle(name):
    case = make_case(name, Nt=8)
    g = case.grid
    eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
    ops = O.Operators(O.Grid(g.mx, g.my), case.kx, case.ky, case.beta, case.gamma)
    V = vectors(g, np.random.default_rng(3))
    dts = np.array([1.0 / 16384, 1.0 / 64, 0.5, 1.0 / 1024])
    got = eng.apply_probe(torch.from_numpy(V).cuda(), torch.from_numpy(dts).cuda()).cpu().numpy()
    for k in range(4):
        ref = ops.step_apply(dts[k], +1, V[k])
        assert rel(got[k], ref) <= 1e-13, (k, rel(got[k], ref))


def test_fft_precond_matches_numpy():
    case = make_case("cfg3", Nt=8)
    g = case.grid
    eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
    dm, dk = tau_diagonals(g, case.beta, case.gamma, case.kx, case.ky)
    Sx, Sy = dst_matrix(g.nx), dst_matrix(g.ny)
    V = vectors(g, np.random.default_rng(4))[:3]
    dts = np.array([1.0 / 16384, 0.25, 1.0 / 64])
    ref = np.stack([(Sy @ ((Sy @ v.reshape(g.ny, g.nx) @ Sx) / (dm + 0.5 * dt * dk)) @ Sx).ravel()
                    for v, dt in zip(V, dts)])
    got = eng.precond_apply(torch.from_numpy(V).cuda(), torch.from_numpy(dts).cuda(), "tau64").cpu().numpy()
    for k in range(3):
        # the DST stages run as FP32 FFTs (the preconditioner only steers the FP64-checked iteration)
        assert rel(got[k], ref[k]) <= 2e-6, (k, rel(got[k], ref[k]))


def test_fft_precond_tensor_core_matches_numpy():
    """The default 'tau' preconditioner of the FFT kernel runs its four DST stages as tcgen05 FP16 GEMMs with the
    DST matrix resident in tensor memory (csrc/rm_tc.cuh): FP16 operands, FP32 accumulation, power-of-two scaling
    by the residual norm -- within 2e-3 of the FP64 preconditioner at every step size, also for inputs 1e+-9 in
    scale (the scaling keeps FP16 in range)."""
    case = make_case("cfg3", Nt=8)
    g = case.grid
    eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
    dm, dk = tau_diagonals(g, case.beta, case.gamma, case.kx, case.ky)
    Sx, Sy = dst_matrix(g.nx), dst_matrix(g.ny)
    V = vectors(g, np.random.default_rng(5))[:3] * np.array([1.0, 1e-9, 1e9])[:, None]
    dts = np.array([1.0 / 16384, 0.25, 1.0 / 64])
    ref = np.stack([(Sy @ ((Sy @ v.reshape(g.ny, g.nx) @ Sx) / (dm + 0.5 * dt * dk)) @ Sx).ravel()
                    for v, dt in zip(V, dts)])
    got = eng.precond_apply(torch.from_numpy(V).cuda(), torch.from_numpy(dts).cuda(), "tau").cpu().numpy()
    for k in range(3):
        assert rel(got[k], ref[k]) <= 2e-3, (k, rel(got[k], ref[k]))


def test_fft_relaxed_precision_applies():
    """'tau' on the FFT kernel applies the operator through FP32 FFTs once |r| <= 1e-6 |b| (rm_sweep.lp_matvec with
    precond 2), 'tau16' keeps every apply in FP64: same iteration count, both accepted on the FP64
    true residual at 1e-12, and the FP32 applies are really used (counter slot 4)."""
    case = make_case("cfg3", Nt=4)
    spec = ProblemSpec(**case.problem_kwargs())
    g = case.grid
    rng = np.random.default_rng(7)
    V = vectors(g, rng)[1:2]                       # a smooth state
    out, its, lowp = {}, {}, {}
    for pre in ("tau", "tau16"):
        disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
        out[pre] = disc.propagate(1.0 / 16384, V)
        its[pre] = int(disc.counters[1].item())
        lowp[pre] = int(disc.counters[4].item())
    assert its["tau"] == its["tau16"] and its["tau"] > 0
    assert lowp["tau"] > 0 and lowp["tau16"] == 0
    assert rel(out["tau"][0], out["tau16"][0]) <= 1e-11
    ops = O.Operators(O.Grid(g.mx, g.my), case.kx, case.ky, case.beta, case.gamma)
    b = ops.step_apply(1.0 / 16384, -1, V[0])
    for pre in out:  # the FP64 true residual of the returned solution
        r = b - ops.step_apply(1.0 / 16384, +1, out[pre][0])
        assert np.linalg.norm(r) <= 1.5e-12 * np.linalg.norm(b), (pre, np.linalg.norm(r) / np.linalg.norm(b))


def test_fft_solve_is_deterministic():
    """Same inputs, same bits: the group reductions are fixed-order and chain results do not depend on which CTA
    group picks a chain up (tools/determinism_check.py runs the long version)."""
    from paper_1805_06688_b200.mgrit import MgritOptions, solve

    case = make_case("cfg3", Nt=256, T=1.0 / 64)
    spec = ProblemSpec(**case.problem_kwargs())
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    U0, t0 = solve(spec, opts, device_result=True)
    U1, t1 = solve(spec, opts, device_result=True)
    assert t0.iterations == t1.iterations and list(t0.cg_iterations) == list(t1.cg_iterations)
    assert torch.equal(U0, U1)


@pytest.mark.parametrize("pre", ["none", "tau", "tau64"])
def test_fft_propagate_matches_oracle(pre):
    case = make_case("cfg3", Nt=4)
    g = case.grid
    spec = ProblemSpec(**case.problem_kwargs())
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-12, preconditioner=pre))
    st = O.Stepper(O.Problem(O.Grid(g.mx, g.my), spec.tmesh.points, case.kx, case.ky, case.beta, case.gamma,
                             spec.source, spec.initial), rel_tol=1e-12)
    V = np.random.default_rng(1).random((3, g.ndof))
    for dt in (1.0 / 16384, 1.0 / 1024, 1.0 / 16):
        got = disc.propagate(dt, V)
        for k in range(3):
            assert rel(got[k], st.propagate(dt, V[k])) <= 1e-10
