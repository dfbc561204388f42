"""Per-point relative L2 distance of GPU MGRIT runs to a reference golden (kept rows exactly, all rows through
the fixed sketches), for several inner solvers / tolerances.

    python tools/parity_scan.py cfg2_full.npz c2f cfg2 [--nt N --T T --M M]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("fixture")
ap.add_argument("tag")
ap.add_argument("config")
ap.add_argument("--nt", type=int, default=None)
ap.add_argument("--T", type=float, default=1.0)
ap.add_argument("--M", type=int, default=None)
a = ap.parse_args()
g = np.load(os.path.join("tests", "golden", a.fixture))
case = make_case(a.config, M=a.M, Nt=a.nt, T=a.T)
spec = ProblemSpec(**case.problem_kwargs())
R = np.random.default_rng(1234).standard_normal((case.grid.ndof, 8)) / np.sqrt(case.grid.ndof)
for pre, tol in (("none", case.cg_rel_tol), ("tau", case.cg_rel_tol), ("tau64", case.cg_rel_tol),
                 ("tau", 1e-13), ("tau", 1e-14), ("none", 1e-14)):
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=tol,
                        cg_preconditioner=pre)
    U, tr = solve(spec, opts)
    keep = [int(k) for k in g[f"{a.tag}_keep"]]
    ek = [np.linalg.norm(U[n] - g[f"{a.tag}_U"][i]) / np.linalg.norm(g[f"{a.tag}_U"][i]) for i, n in enumerate(keep)]
    S = U @ R
    es = np.linalg.norm(S - g[f"{a.tag}_sketch"], axis=1) / (np.linalg.norm(g[f"{a.tag}_sketch"], axis=1) + 1e-300)
    print(f"{pre:5s} tol={tol:g} its={tr.iterations}: kept max {max(ek):.2e} at {keep[int(np.argmax(ek))]}; "
          f"sketch max {es.max():.2e} at {int(es.argmax())}, median {np.median(es):.2e}; kept {['%.1e' % e for e in ek]}",
          flush=True)
