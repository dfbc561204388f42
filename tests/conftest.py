import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU oracle checks")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))
        return cache[name]

    return load


@pytest.fixture
def rng():
    return np.random.default_rng(42)


def manufactured(beta=0.8, gamma=0.7, kx=2.0, ky=0.5):
    """The reference's manufactured Example 4.1 (verify.py:28-70), restated for the tests."""
    import math

    def exact(x, y, t):
        return 10.0 * np.exp(-t) * (x - x**2) ** 2 * (y - y**2) ** 2

    def bracket(s, order):
        g3, g4, g5 = (math.gamma(k - 2.0 * order) for k in (3.0, 4.0, 5.0))
        p2, p3, p4 = 2.0 - 2.0 * order, 3.0 - 2.0 * order, 4.0 - 2.0 * order
        return ((s**p2 + (1.0 - s) ** p2) / g3 - 6.0 * (s**p3 + (1.0 - s) ** p3) / g4
                + 12.0 * (s**p4 + (1.0 - s) ** p4) / g5)

    def source(x, y, t):
        x = np.asarray(x, dtype=float)
        y = np.asarray(y, dtype=float)
        d = 10.0 * np.exp(-t)
        wx, wy = (x - x**2) ** 2, (y - y**2) ** 2
        out = -d * wx * wy
        out = out + d * kx * wy / math.cos(beta * math.pi) * bracket(x, beta)
        out = out + d * ky * wx / math.cos(gamma * math.pi) * bracket(y, gamma)
        return out

    def initial(x, y):
        return exact(x, y, 0.0)

    return dict(beta=beta, gamma=gamma, kx=kx, ky=ky, source=source, initial=initial, exact=exact)
