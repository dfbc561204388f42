"""Per-phase cycles of the FFT chain kernel's PCG iteration (CTA 0), from the -DRM_TIMING library:

    python -c "from paper_1805_06688_b200 import build; build.build(timing=True)"
    RM_LIB=paper_1805_06688_b200/_lib/libriesz_mgrit_b200_timing.so python tools/fft_phase_timing.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.engine import Engine  # noqa: E402

NAMES = ["apply: column pass", "apply: group barrier", "apply: row pass + combine", "reduce p.Ap",
         "(unused)", "precond: row DST", "precond: barrier 1", "precond: column DSTs", "precond: barrier 2",
         "precond: row DST (inverse)", "reduce r.r, r.z", "x/p update + barrier"]


def main():
    case = make_case("cfg3", Nt=8)
    eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
    n = case.grid.ndof
    nch, m = 18, 4
    N = nch * m
    U = torch.from_numpy(np.random.default_rng(0).random((N + 1, n))).cuda()
    G_ = torch.zeros_like(U)
    dt = torch.full((N,), 1.0 / 16384, dtype=torch.float64, device="cuda")
    for rep in range(2):
        cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
        t0 = (ctypes.c_longlong * 16)()
        torch.cuda.synchronize()
        eng.lib.rm_debug_timing(eng.handle, t0)
        V = U.clone()
        eng.sweep(nchains=nch, first=1, cstride=m, clen=m - 1, nmax=N, dt=dt, counters=cnt, rel_tol=1e-12,
                  src=V, x0_mode=1, gadd=G_, out=V, precond="tau")
        torch.cuda.synchronize()
        t1 = (ctypes.c_longlong * 16)()
        eng.lib.rm_debug_timing(eng.handle, t1)
    c = cnt.cpu().tolist()
    its = c[1] / max(nch, 1)  # per chain (CTA 0 runs about one chain's share)
    d = np.array(t1[:]) - np.array(t0[:])
    tot = d.sum()
    print(f"solves={c[0]} its={c[1]} applies={c[2]} precond={c[3]}; CTA0 cycles total {tot}")
    for k, name in enumerate(NAMES):
        if d[k]:
            print(f"  {name:28s} {d[k]:12d} cycles  {100 * d[k] / tot:5.1f}%")


if __name__ == "__main__":
    main()
