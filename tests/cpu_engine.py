"""TEST INFRASTRUCTURE: a CPU stand-in for the device engine, built on the oracle.

It implements the ``Engine.sweep`` contract (include/riesz_mgrit_b200.h, rm_sweep)
with the oracle's operators and CG so that the host-side MGRIT orchestration --
in particular the multi-rank time-slab logic (timeslab.py, gloo backend) -- can
be exercised on a machine without a GPU.  The product never constructs it.
"""

import numpy as np
import torch

from oracle import riesz_oracle as O
from paper_1805_06688_b200.krylov import CgFailure
from paper_1805_06688_b200.stepper import DeviceLoads


def _row(a, n):
    if isinstance(a, tuple):
        t, off = a
        return t[n + off]
    return a[n]


class CpuEngine:
    def __init__(self, grid, beta, gamma, kx, ky):
        self.ops = O.Operators(O.Grid(grid.mx, grid.my), kx, ky, beta, gamma)
        self.ndof = grid.ndof
        self.launches = 0
        self.fail = None

    def sweep(self, *, nchains, first, cstride, clen, nmax, dt, counters, rel_tol, src=None, explicit=True,
              x0_mode=1, x0=None, f=None, f_stride=0, fscale=None, gadd=None, sub=None, out=None, out_div=1,
              norms=None, max_iter=None, group=0, row=None, tag="", precond="none", guess=None, keep=None,
              hg=None, ax=None, gax=None, ain=None):
        self.launches += 1
        for c in range(nchains):
            n0 = first + c * cstride
            n1 = min(n0 + clen - 1, nmax)
            for n in range(n0, n1 + 1):
                h = float(_row(dt, n - 1))
                vin = (_row(src, n - 1) if n == n0 else _row(out, n - 1)).numpy() if (explicit or x0_mode == 1) else None
                b = np.zeros(self.ndof)
                if explicit:
                    b = self.ops.step_apply(h, -1, vin)
                if f is not None:
                    fr = (_row(f, 0) if f_stride == 0 else _row(f, n)).numpy()
                    fs = float(_row(fscale, n)) if fscale is not None else 1.0
                    b = fs * fr + b if explicit else fs * fr
                start = vin if x0_mode == 1 else (_row(x0, n).numpy() if x0_mode == 2 else None)
                try:
                    x, its = O.cg(lambda v: self.ops.step_apply(h, +1, v), b, x0=start, rel_tol=rel_tol,
                                  max_iter=max_iter)
                except O.OracleCgFailure as exc:
                    if self.fail is None:
                        self.fail = (n, exc)
                    counters += torch.tensor([1, exc.iterations, 0, 0, 0])
                    break
                counters += torch.tensor([1, its, its + 2, 0, 0])
                y = x
                if gadd is not None:
                    y = _row(gadd, n).numpy() + y
                if keep is not None:
                    _row(keep, n // out_div).copy_(torch.from_numpy(y))
                if sub is not None:
                    y = y - _row(sub, n).numpy()
                if out is not None:
                    _row(out, n // out_div).copy_(torch.from_numpy(y))
                if norms is not None:
                    _row(norms, n // out_div).fill_(float(y @ y))

    def check_fail(self):
        if self.fail is not None:
            n, exc = self.fail
            self.fail = None
            raise CgFailure(f"CG failure at time index {n}", exc.residual_norm, exc.iterations)

    def correct(self, U, Uc, m):
        for k in range(Uc.shape[0]):
            U[k * m] += Uc[k]

    def diff_sqnorm(self, a, b, out):
        d = (a - b).numpy()
        out[0] = float(d @ d)

    def pcg64_fill(self, seed, out, start=0):
        rng = np.random.default_rng(seed)
        rng.bit_generator.advance(start)
        out.copy_(torch.from_numpy(rng.random(out.numel()).reshape(out.shape)))


class CpuDisc:
    """Minimal Discretization stand-in used through MgritHierarchy(disc_factory=...)."""

    def __init__(self, spec, cg_opts, engine=None):
        self.spec = spec
        self.cg_opts = cg_opts
        self.engine = engine or CpuEngine(spec.grid, spec.beta, spec.gamma, spec.kx, spec.ky)
        self.device = torch.device("cpu")
        self.counters = torch.zeros(5, dtype=torch.int64)
        self.ndof = spec.grid.ndof

    def device_loads(self, points):
        prob = O.Problem(O.Grid(self.spec.grid.mx, self.spec.grid.my), points, self.spec.kx, self.spec.ky,
                         self.spec.beta, self.spec.gamma, self.spec.source, self.spec.initial)
        st = O.Stepper(prob)
        F = np.zeros((points.size, self.ndof))
        for n in range(1, points.size):
            F[n] = st.load(n)
        return DeviceLoads(torch.from_numpy(F), self.ndof, None)


def cpu_disc_factory(spec, cg_opts, engine):
    return CpuDisc(spec, cg_opts, engine)
