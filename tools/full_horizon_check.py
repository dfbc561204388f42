"""Full-size run of a config with the default solver against the reference-algorithm path ('none': the reference's
unpreconditioned CG with its exact stopping rule, pinned to the reference's own runs in tests/test_gpu_regimes.py):
per-time-point relative L2 distance, iteration counts and times.

    python tools/full_horizon_check.py [--config cfg3] [--solvers tau tau64]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--nt", type=int, default=None)
ap.add_argument("--solvers", nargs="+", default=["tau", "tau64"])
a = ap.parse_args()
case = make_case(a.config, Nt=a.nt)
spec = ProblemSpec(**case.problem_kwargs())


def run(pre):
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol,
                        cg_preconditioner=pre)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    U, tr = solve(spec, opts, device_result=True)
    torch.cuda.synchronize()
    return U, tr, time.perf_counter() - t0


Uref, tref, sref = run("none")
nref = torch.linalg.norm(Uref, dim=1).clamp_min(1e-300)
print(f"none : its={tref.iterations} solves={tref.spatial_solves[-1]} cg={tref.cg_iterations[-1]} {sref:.1f} s "
      f"residuals {[f'{r:.3e}' for r in tref.residual_norms]}")
for pre in a.solvers:
    U, tr, s = run(pre)
    e = torch.linalg.norm(U - Uref, dim=1) / nref
    print(f"{pre:5s}: its={tr.iterations} solves={tr.spatial_solves[-1]} cg={tr.cg_iterations[-1]} {s:.1f} s; per-point "
          f"rel. L2 vs 'none': max {e.max().item():.2e} at n={int(e.argmax())}, median {e.median().item():.2e}")
    del U
