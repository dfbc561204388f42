"""Pin the CPU oracle (oracle/riesz_oracle.py) to golden vectors produced by the reference.

CPU only.  The oracle is the checker of the GPU parity tests and the timed CPU
implementation of bench.py's reference arm, so it must reproduce the
reference's own outputs first.
"""

import numpy as np
import pytest

from conftest import manufactured
from oracle import riesz_oracle as O
from paper_1805_06688_b200.configs import make_case


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def man_problem(M, N, **kw):
    c = manufactured(**kw)
    return O.Problem(O.Grid(M, M), O.uniform_points(1.0, N), c["kx"], c["ky"], c["beta"], c["gamma"],
                     c["source"], c["initial"])


def case_problem(case):
    return O.Problem(O.Grid(case.grid.mx, case.grid.my), case.tmesh.points, case.kx, case.ky, case.beta,
                     case.gamma, case.source, case.initial)


@pytest.mark.parametrize("case", range(5))
def test_operators(golden, case):
    g = golden("operators.npz")
    mx, my, b, gm, kx, ky = g[f"c{case}_params"]
    ops = O.Operators(O.Grid(int(mx), int(my)), kx, ky, b, gm)
    V = g[f"c{case}_v"]
    for k in range(V.shape[0]):
        assert np.array_equal(ops.mass(V[k]), g[f"c{case}_mass"][k])
        assert np.array_equal(ops.sx(V[k]), g[f"c{case}_sx"][k])
        assert np.array_equal(ops.sy(V[k]), g[f"c{case}_sy"][k])
        dt = g[f"c{case}_dts"][k]
        assert np.array_equal(ops.step_apply(dt, +1, V[k]), g[f"c{case}_imp"][k])
        assert np.array_equal(ops.step_apply(dt, -1, V[k]), g[f"c{case}_exp"][k])
    a, c, r = O.stiffness_gens(int(mx), b)
    assert np.array_equal(a, g[f"c{case}_a1"])
    assert np.array_equal(c, g[f"c{case}_a2col"])
    assert np.array_equal(r, g[f"c{case}_a2row"])


@pytest.mark.parametrize("k", range(4))
def test_cg(golden, k):
    g = golden("cg.npz")
    M, dt, warm, tol = g[f"k{k}_params"]
    c = manufactured(0.6, 0.7, 2.0, 0.5)
    ops = O.Operators(O.Grid(int(M), int(M)), c["kx"], c["ky"], c["beta"], c["gamma"])
    x, its = O.cg(lambda v: ops.step_apply(dt, +1, v), g[f"k{k}_b"], x0=g[f"k{k}_x0"] if warm else None,
                  rel_tol=tol)
    assert its == int(g[f"k{k}_its"])
    assert np.array_equal(x, g[f"k{k}_x"])


def test_stepper(golden):
    g = golden("stepper.npz")
    prob = man_problem(4, 8)
    st = O.Stepper(prob, rel_tol=1e-13)
    assert np.array_equal(np.stack([st.load(n) for n in range(1, 9)]), g["loads"])
    assert np.array_equal(np.stack([st.g_vector(n) for n in range(1, 9)]), g["gvecs"])
    assert np.array_equal(st.propagate(0.125, g["prop_v"]), g["prop_out"])
    assert np.array_equal(O.sequential(prob, O.Stepper(prob, rel_tol=1e-13)), g["seq"])
    U = g["seq"].copy()
    U[3] += 1e-3
    norms, tot = O.spacetime_residual(prob, U, O.Stepper(prob, rel_tol=1e-13))
    assert np.array_equal(norms, g["stres_norms"])
    assert tot == float(g["stres_total"])


RUNS = {
    "two": dict(m=4, max_levels=2),
    "multi": dict(m=4),
    "noskip": dict(m=4, skip_first_down=False),
    "frelax": dict(m=2, relaxation="f"),
    "seed3": dict(m=8, rng_seed=3),
}


@pytest.mark.parametrize("tag", list(RUNS))
def test_mgrit_small(golden, tag):
    g = golden("mgrit_small.npz")
    U, tr = O.mgrit_solve(man_problem(8, 64), O.Options(halt_tol=1e-10, cg_rel_tol=1e-12, **RUNS[tag]))
    assert np.array_equal(U, g[f"{tag}_U"])
    assert tr.residual_norms == list(g[f"{tag}_res"])
    assert tr.spatial_solves == list(g[f"{tag}_solves"])
    assert tr.cg_iterations == list(g[f"{tag}_cgits"])


def test_parareal_small(golden):
    g = golden("mgrit_small.npz")
    U, tr = O.parareal(man_problem(8, 64), O.Options(m=8, halt_tol=1e-10, cg_rel_tol=1e-12))
    assert np.array_equal(U, g["parareal_U"])
    assert tr.residual_norms == list(g["parareal_res"])


def test_cfg1_two_level(golden):
    """The BASELINE config-1 run (about 10 s of numpy)."""
    g = golden("cfg1.npz")
    case = make_case("cfg1")
    U, tr = O.mgrit_solve(case_problem(case), O.Options(m=4, max_levels=2, halt_tol=1e-8, cg_rel_tol=1e-12))
    assert tr.iterations == 13
    assert np.array_equal(U, g["two_U"])
    assert tr.residual_norms == list(g["two_res"])


def test_reduced_graded(golden):
    g = golden("reduced.npz")
    case = make_case("cfg4", M=16, Nt=64)
    U, tr = O.mgrit_solve(case_problem(case), O.Options(m=8, max_levels=2, halt_tol=1e-8, cg_rel_tol=1e-12))
    assert np.array_equal(U, g["g_two_U"])
    assert tr.spatial_solves == list(g["g_two_solves"])


def test_pcg64_restatement(golden):
    g = golden("pcg64.npz")
    s, inc = O.pcg64_state(0)
    assert (hex(s), hex(inc)) == tuple(g["state_hex"])
    assert np.array_equal(O.pcg64_uniform(0, 0, 16), g["first"])
    for off, val in zip(g["offsets"], g["values"]):
        assert O.pcg64_uniform(0, int(off), 1)[0] == val
