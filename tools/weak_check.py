"""MGRIT iteration counts and time-to-solution of cfg2-sized families on one GPU (weak-scaling study).

    python tools/weak_check.py          # Nt = 4096 k at T = 1 (finer steps): 8 MGRIT iterations for k = 2, 8
    python tools/weak_check.py horizon  # Nt = 4096 k at T = k (same step, longer horizon): 30 / 90 iterations
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

horizon = len(sys.argv) > 1 and sys.argv[1] == "horizon"
for k in (1, 2, 8):
    T = float(k) if horizon else 1.0
    case = make_case("cfg2", Nt=4096 * k, T=T)
    spec = ProblemSpec(**case.problem_kwargs())
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U, tr = solve(spec, opts, device_result=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"Nt={4096 * k} T={T:g}: iters={tr.iterations} TTS={t:.3f}s per-4096-block={t / k:.3f}s "
          f"res={tr.residual_norms[-1]:.2e}", flush=True)
