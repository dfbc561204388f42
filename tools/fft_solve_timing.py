"""Solve-level cycles of the FFT chain kernel (CTA 0) over the level-0 F-relaxation of cfg3's initial residual, from a
-DRM_TIMING,RM_TIMING_SOLVE build:

    RM_DEFINES=RM_TIMING_SOLVE RM_LIB_OUT=/path/lib_solve.so python -c "from paper_1805_06688_b200 import build; build.build(timing=True, force=True)"
    RM_LIB=/path/lib_solve.so python tools/fft_solve_timing.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.engine import Engine  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

NAMES = ["step prologue (rhs, initial residual, second guess)", "first direction (precond + publish)",
         "PCG iterations", "acceptance (x update, true-residual apply)", "epilogue (store, norms, barriers)",
         "  prologue: chain input + barrier", "  prologue: mass stencil of the step input",
         "  prologue: right-hand side (apply or apply-free), stores", "  prologue: reduce |b|, |r0|"]
case = make_case("cfg3", Nt=4096, T=0.25)
eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
spec = ProblemSpec(**case.problem_kwargs())
solve(spec, opts, device_result=True, engine=eng)
torch.cuda.synchronize()
t0 = (ctypes.c_longlong * 16)()
eng.lib.rm_debug_timing(eng.handle, t0)
_, tr = solve(spec, opts, device_result=True, engine=eng)
torch.cuda.synchronize()
t1 = (ctypes.c_longlong * 16)()
eng.lib.rm_debug_timing(eng.handle, t1)
d = np.array(t1[:]) - np.array(t0[:])
tot = d[:5].sum()
print(f"iterations={tr.iterations} solves={tr.spatial_solves[-1]} cg={tr.cg_iterations[-1]}; CTA 0 cycles {tot}")
d[0] = d[0] + d[5:9].sum()  # (the sub-slots split the prologue; the rest of it is the second guess)
tot = d[:5].sum()
for k, name in enumerate(NAMES):
    print(f"  {name:55s} {d[k]:14d} cycles {100 * d[k] / tot:5.1f}%")
