"""theory.two_level_bound (reference theory.py:88-134) against the reference's own values (tests/golden/theory.npz),
and the predicted-vs-observed comparison the reference's factor studies make (verify.py:208-251)."""

import numpy as np
import pytest

from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.stepper import ProblemSpec
from paper_1805_06688_b200.theory import mode_spectrum, step_factors, two_level_bound


@pytest.mark.parametrize("tag,name,kw,m", [("t1", "cfg1", {}, 4), ("t2", "cfg2", dict(M=32, Nt=512), 8),
                                           ("t4", "cfg4", dict(M=64, Nt=512), 8)])
def test_two_level_bound_matches_reference(golden, tag, name, kw, m):
    g = golden("theory.npz")
    case = make_case(name, **kw)
    spec = ProblemSpec(**case.problem_kwargs())
    sp = mode_spectrum(spec)
    np.testing.assert_allclose(sp.sigmas, g[f"{tag}_sigmas"], rtol=1e-9)
    rep = two_level_bound(sp, spec.tmesh, m)
    assert rep.bound == pytest.approx(float(g[f"{tag}_bound"]), rel=1e-8)
    assert rep.argmax_mode == int(g[f"{tag}_argmax"])
    np.testing.assert_allclose(rep.per_mode, g[f"{tag}_per_mode"], rtol=1e-7, atol=1e-14)


def test_step_factors_range():
    s = np.array([1e-3, 1.0, 1e3, 1e9])
    f = step_factors(s, 0.5)
    assert np.all(np.abs(f) < 1.0) and f[0] > 0.99 and f[-1] < -0.99


def test_predicted_vs_observed_cfg1(golden):
    """cfg1 two-level (m = 4): the bound (0.232) holds the observed asymptotic factor of the reference's own run;
    the cfg4 physics' bound exceeds 1, matching the divergence of the reference's MGRIT there."""
    g = golden("theory.npz")
    res = golden("cfg1.npz")["two_res"]
    observed = (res[-1] / res[-6]) ** 0.2
    assert observed <= float(g["t1_bound"])
    assert float(g["t4_bound"]) > 1.0
    div = golden("cfg4_diverge.npz")["c4d_res"]
    assert np.all(np.diff(div) > 0)
