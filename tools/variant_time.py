"""Developer tool: time the cfg3 solve with the library named by RM_LIB (variants built by tools/build_variant.sh).

    RM_LIB=paper_1805_06688_b200/_lib/var_X.so RM_NO_BUILD=1 python tools/variant_time.py [repeats]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.engine import Engine  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402

rep = int(sys.argv[1]) if len(sys.argv) > 1 else 3
case = make_case("cfg3")
spec = ProblemSpec(**case.problem_kwargs())
opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
ts = []
for i in range(rep):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    U, tr = solve(spec, opts, device_result=True, engine=eng)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(os.environ.get("RM_LIB", "default"), "times", [round(t, 3) for t in ts], "min", round(min(ts[1:] or ts), 3),
      "its", tr.iterations, "solves", sum(tr.spatial_solves), "cg", sum(tr.cg_iterations),
      "res", f"{tr.residual_norms[-1]:.6e}", "unorm", f"{float(U.norm()):.15e}")
