"""MGRIT residual history of one configuration on the GPU (prints the trace even when the solve fails).

    python tools/residual_history.py --config cfg4 [--M 512] [--nt 8192] [--levels 2|none] [--iters 6]
"""

import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritFailure, MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--levels", default="default")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--precond", default="tau")
    ap.add_argument("--T", type=float, default=1.0)
    a = ap.parse_args()
    case = make_case(a.config, M=a.M, Nt=a.nt, T=a.T)
    lv = case.max_levels if a.levels == "default" else (None if a.levels == "none" else int(a.levels))
    opts = MgritOptions(m=case.m, max_levels=lv, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol,
                        max_iters=a.iters, cg_preconditioner=a.precond)
    t0 = time.perf_counter()
    try:
        _, tr = solve(ProblemSpec(**case.problem_kwargs()), opts, device_result=True)
        status = "converged"
    except MgritFailure as exc:
        tr = exc.trace
        status = "not converged"
    torch.cuda.synchronize()
    print(f"{case.name} M={case.grid.mx} Nt={case.tmesh.n_intervals} levels={lv} precond={a.precond}: {status} "
          f"after {tr.iterations} its, {time.perf_counter() - t0:.1f}s; residuals "
          + " ".join("%.3e" % r for r in tr.residual_norms), flush=True)


if __name__ == "__main__":
    main()
