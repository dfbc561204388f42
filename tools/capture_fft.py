"""One cfg3 solve for ncu: the first chain_fft_kernel launch of the process is the level-0 F-relaxation of the initial
residual (1024 chains x 15 steps on the random initial guess).

    ncu --set full -k regex:chain_fft --launch-count 1 -o out python tools/capture_fft.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

case = make_case("cfg3")
opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, max_iters=1)
try:
    solve(ProblemSpec(**case.problem_kwargs()), opts, device_result=True)
except Exception as exc:  # one cycle is enough (MgritFailure)
    print(type(exc).__name__)
torch.cuda.synchronize()
