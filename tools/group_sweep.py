"""Time one F-relaxation-shaped sweep (chains of m-1 steps) for each cluster size G."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.engine import Engine

case = make_case("cfg2", Nt=8)
eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
n = case.grid.ndof
for nch, dtv in ((512, 1 / 4096), (64, 1 / 512), (8, 1 / 64), (1, 1 / 8)):
    N = nch * 8
    U = torch.from_numpy(np.random.default_rng(0).random((N + 1, n))).cuda()
    G_ = torch.zeros_like(U)
    dt = torch.full((N,), dtv, dtype=torch.float64, device="cuda")
    for pre in ("tau",):
        res = []
        for Gs in (1, 2, 4, 8, 16):
            try:
                cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
                V = U.clone()
                eng.sweep(nchains=nch, first=1, cstride=8, clen=7, nmax=N, dt=dt, counters=cnt, rel_tol=1e-12,
                          src=V, x0_mode=1, gadd=G_, out=V, group=Gs, precond=pre)
                torch.cuda.synchronize()
                V = U.clone()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                cnt.zero_()
                e0.record()
                eng.sweep(nchains=nch, first=1, cstride=8, clen=7, nmax=N, dt=dt, counters=cnt, rel_tol=1e-12,
                          src=V, x0_mode=1, gadd=G_, out=V, group=Gs, precond=pre)
                e1.record()
                torch.cuda.synchronize()
                c = cnt.cpu().tolist()
                res.append(f"G={Gs}: {e0.elapsed_time(e1):7.2f} ms ({c[1] / max(c[0], 1):.1f} its)")
            except Exception as ex:
                res.append(f"G={Gs}: n/a")
        print(f"chains={nch:4d} dt={dtv:.2e} {pre}: " + "  ".join(res))
