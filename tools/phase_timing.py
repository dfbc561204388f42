"""Per-phase cycle breakdown of the CG loop (needs the -DRM_TIMING library: RM_LIB=..._timing.so)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.engine import Engine  # noqa: E402

NAMES = ["matvec", "Ap+pAp partial", "reduce pAp", "x/r update", "reduce rr(+rz)", "p update", "sync p", "loop top",
         "tau: r->tile", "tau: dst_x", "tau: x->tile", "tau: dst_y", "tau: scale->tile"]


PRE = os.environ.get('RM_PRECOND', 'tau')


def main():
    case = make_case("cfg2", Nt=8)
    eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
    n = case.grid.ndof
    for G, B in ((2, 512), (4, 512), (8, 64), (16, 8)):
        V = torch.from_numpy(np.random.default_rng(0).random((B, n))).cuda()
        dt = torch.full((B,), 1.0 / 4096, dtype=torch.float64, device="cuda")
        out = torch.empty_like(V)
        cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
        zero = (ctypes.c_longlong * 16)()
        eng.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dt, counters=cnt, rel_tol=1e-12, src=V,
                  x0_mode=1, out=(out, -1), group=G, precond=PRE)
        torch.cuda.synchronize()
        t0 = (ctypes.c_longlong * 16)()
        eng.lib.rm_debug_timing(eng.handle, t0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cnt.zero_()
        e0.record()
        eng.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dt, counters=cnt, rel_tol=1e-12, src=V,
                  x0_mode=1, out=(out, -1), group=G, precond=PRE)
        e1.record()
        torch.cuda.synchronize()
        t1 = (ctypes.c_longlong * 16)()
        eng.lib.rm_debug_timing(eng.handle, t1)
        d = [t1[i] - t0[i] for i in range(13)]
        c = cnt.cpu().tolist()
        its_cta0 = None
        tot = sum(d)
        print(f"G={G} B={B}: {e0.elapsed_time(e1):.2f} ms, solves={c[0]} cg={c[1]} mv={c[2]}; CTA0 cycles by phase:")
        for name, v in zip(NAMES, d):
            print(f"   {name:16s} {v:12d}  {100 * v / max(tot, 1):5.1f}%")
        del its_cta0


if __name__ == "__main__":
    main()
