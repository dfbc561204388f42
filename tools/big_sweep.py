"""Throughput of the large-grid chain kernel: one F-relaxation-shaped sweep (chains of m-1 steps).

    python tools/big_sweep.py [--config cfg3|cfg4] [--chains 64] [--steps 7]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.engine import Engine  # noqa: E402
from paper_1805_06688_b200.flops import fmv, fpc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--chains", type=int, nargs="+", default=[37, 148])
ap.add_argument("--steps", type=int, default=7)
ap.add_argument("--dt", type=float, default=None)
ap.add_argument("--precond", default="tau")
a = ap.parse_args()
case = make_case(a.config, Nt=8)
eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)
n = case.grid.ndof
dtv = a.dt or 1.0 / (case.tmesh.n_intervals if a.dt else 16384)
F, FP = fmv(case.grid.nx, case.grid.ny, eng.flags), fpc(case.grid.nx, case.grid.ny)
for nch in a.chains:
    m = a.steps + 1
    N = nch * m
    U = torch.from_numpy(np.random.default_rng(0).random((N + 1, n))).cuda()
    G_ = torch.zeros_like(U)
    dt = torch.full((N,), dtv, dtype=torch.float64, device="cuda")
    for rep in range(2):
        cnt = torch.zeros(5, dtype=torch.int64, device="cuda")
        V = U.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.sweep(nchains=nch, first=1, cstride=m, clen=m - 1, nmax=N, dt=dt, counters=cnt, rel_tol=1e-12,
                  src=V, x0_mode=1, gadd=G_, out=V, precond=a.precond)
        e1.record()
        torch.cuda.synchronize()
        c = cnt.cpu().tolist()
        ms = e0.elapsed_time(e1)
        tf = (c[2] * F + c[3] * FP) / (ms * 1e-3) / 1e12
        print(f"{a.config} {a.precond} chains={nch} steps={m - 1}: {ms:8.2f} ms, {c[1] / max(c[0], 1):.1f} its/solve, "
              f"{c[2]} applies, {c[3]} precond -> {tf:.2f} TF/s", flush=True)
