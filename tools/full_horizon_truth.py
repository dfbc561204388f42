"""Distance of full-size runs (inner tolerance 1e-12) to the converged answer (inner tolerance 1e-13, reference
algorithm; 1e-14 is below what FP64 CG attains on these right-hand sides), per time point: which of two correct inner solvers is closer to the truth over a long horizon.

    python tools/full_horizon_truth.py [--config cfg3]
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
ap.add_argument("--nt", type=int, default=None)
a = ap.parse_args()
case = make_case(a.config, Nt=a.nt)
spec = ProblemSpec(**case.problem_kwargs())


def run(pre, tol):
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=tol,
                        cg_preconditioner=pre)
    U, tr = solve(spec, opts, device_result=True)
    torch.cuda.synchronize()
    return U, tr


T, tt = run("none", 1e-13)
nT = torch.linalg.norm(T, dim=1).clamp_min(1e-300)
print(f"truth (none @ 1e-13): its={tt.iterations}")
for pre, tol in (("none", 1e-12), ("tau", 1e-12), ("tau64", 1e-12), ("tau", 1e-13)):
    U, tr = run(pre, tol)
    e = torch.linalg.norm(U - T, dim=1) / nT
    print(f"{pre:5s} @ {tol:g}: its={tr.iterations}; per-point rel. L2 to the truth: max {e.max().item():.2e}, "
          f"median {e.median().item():.2e}", flush=True)
    del U
