"""Where the end-to-end (public API, host result) time of one cfg2 solve goes.

    python tools/e2e_breakdown.py [--config cfg2]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.engine import Engine  # noqa: E402
from paper_1805_06688_b200.mgrit import MgritOptions, solve  # noqa: E402
from paper_1805_06688_b200.stepper import ProblemSpec  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    a = ap.parse_args()
    case = make_case(a.config)
    spec = ProblemSpec(**case.problem_kwargs())
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    for rep in range(3):
        t0 = t()
        eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
        eng.ensure_tau()
        t1 = t()
        U, tr = solve(spec, opts, device_result=True, engine=eng)
        t2 = t()
        Uh = U.cpu().numpy()
        t3 = t()
        pin = torch.empty(U.shape, dtype=U.dtype, pin_memory=True)
        t4 = t()
        pin.copy_(U)
        t5 = t()
        Uf, tr = solve(spec, opts)
        t6 = t()
        print(f"rep {rep}: engine+tau {1e3*(t1-t0):.1f} ms | solve(device) {1e3*(t2-t1):.1f} ms | "
              f"d2h pageable {1e3*(t3-t2):.1f} ms ({Uh.nbytes/1e6:.0f} MB) | pinned alloc {1e3*(t4-t3):.1f} ms | "
              f"d2h pinned {1e3*(t5-t4):.1f} ms | public solve() {1e3*(t6-t5):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
