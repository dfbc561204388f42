"""Run the same MGRIT solve several times on the GPU and compare results bitwise (and the work counters).

    python tools/determinism_check.py [--config cfg3] [--nt 2048] [--runs 3] [--precond tau]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--nt", type=int, default=2048)
ap.add_argument("--T", type=float, default=0.125)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--precond", default="tau")
a = ap.parse_args()
case = make_case(a.config, Nt=a.nt, T=a.T)
spec = ProblemSpec(**case.problem_kwargs())
opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol,
                    cg_preconditioner=a.precond)
ref = None
for r in range(a.runs):
    U, tr = solve(spec, opts, device_result=True)
    torch.cuda.synchronize()
    tot = (tr.iterations, tr.spatial_solves[-1], tr.cg_iterations[-1])
    if ref is None:
        ref = (U.clone(), tot)
        print("run 0:", tot)
    else:
        same = bool(torch.equal(U, ref[0]))
        print(f"run {r}: {tot} bitwise_equal={same} max|diff|={(U - ref[0]).abs().max().item():.3e}")
