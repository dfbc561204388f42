"""TEST INFRASTRUCTURE: a CPU stand-in for the device engine, built on the oracle.

It implements the ``Engine.sweep`` contract (include/riesz_mgrit_b200.h, rm_sweep) with the oracle's operators
and CG -- including the reuse inputs of the device kernels (second starting guess ``guess``/``gax``, apply-free
right-hand sides from ``hg``/``ain``, stored ``A x`` rows ``ax``, kept C-point values ``keep``) -- so that the
host-side MGRIT orchestration, in particular the multi-rank time-slab logic (timeslab.py, gloo backend) and the
slab-local row offsets of every array it passes, can be exercised on a machine without a GPU.  The product
never constructs it.
"""

import numpy as np
import torch

from oracle import riesz_oracle as O
from paper_1805_06688_b200.krylov import CgFailure
from paper_1805_06688_b200.stepper import DeviceLoads


def _row(a, n):
    """Row n (a global time index) of a sweep array: a tensor, or (tensor, offset) as Engine.sweep takes it."""
    if isinstance(a, tuple):
        t, off = a
        i = n + off
    else:
        t, i = a, n
    if not 0 <= i < t.shape[0]:
        raise IndexError(f"row {n} outside the array passed to the sweep (local index {i} of {t.shape[0]})")
    return t[i]


class CpuEngine:
    apply = True  # marks an engine with operator applies: the host then keeps the apply-reuse rows (HG, AX)

    def __init__(self, grid, beta, gamma, kx, ky):
        self.ops = O.Operators(O.Grid(grid.mx, grid.my), kx, ky, beta, gamma)
        self.ndof = grid.ndof
        self.launches = 0
        self.fail = None

    def _A(self, h, v):
        return self.ops.step_apply(h, +1, v)

    def sweep(self, *, nchains, first, cstride, clen, nmax, dt, counters, rel_tol, src=None, explicit=True,
              x0_mode=1, x0=None, f=None, f_stride=0, fscale=None, gadd=None, sub=None, out=None, out_div=1,
              norms=None, max_iter=None, group=0, row=None, tag="", precond="none", guess=None, keep=None,
              hg=None, ax=None, gax=None, ain=None, gscale=None):
        self.launches += 1

        def grow(a, n):  # row n of G or A G (a single vector times gscale[n] when compressed)
            return float(gscale[n]) * a.numpy() if gscale is not None else _row(a, n).numpy()

        need_in = explicit or x0_mode == 1
        for c in range(nchains):
            n0 = first + c * cstride
            n1 = min(n0 + clen - 1, nmax)
            prev = None  # (s, b, r) of the previous accepted solve of this chain
            for n in range(n0, n1 + 1):
                h = float(_row(dt, n - 1))
                s = 0.5 * h
                in_tile = n > n0
                vin = (_row(src, n - 1) if not in_tile else _row(out, n - 1)).numpy() if need_in else None
                b = np.zeros(self.ndof)
                if explicit:
                    free = in_tile and prev is not None and hg is not None and gadd is not None and sub is None
                    use_ain = not in_tile and n >= 2 and ain is not None and hg is not None
                    if free:  # (M - s K) y = (1 + s/s0) M y - (s/s0)(b - r + A_{s0} G_{n-1})
                        s0, bp, rp = prev
                        q = s / s0
                        b = (1 + q) * self.ops.mass(vin) - q * (bp - rp + grow(hg, n - 1))
                    elif use_ain:
                        q = s / (0.5 * float(_row(dt, n - 2)))
                        b = (1 + q) * self.ops.mass(vin) - q * (_row(ain, n - 1).numpy() + grow(hg, n - 1))
                    else:
                        b = self.ops.step_apply(h, -1, vin)
                if f is not None:
                    fr = (_row(f, 0) if f_stride == 0 else _row(f, n)).numpy()
                    fs = float(_row(fscale, n)) if fscale is not None else 1.0
                    b = fs * fr + b if explicit else fs * fr
                start = vin if x0_mode == 1 else (_row(x0, n).numpy() if x0_mode == 2 else np.zeros(self.ndof))
                target = rel_tol * np.linalg.norm(b) if np.linalg.norm(b) > 0 else rel_tol
                r0 = b - self._A(h, start)
                if guess is not None and x0_mode < 3 and np.linalg.norm(r0) > target:
                    g2 = _row(guess, n).numpy() - (grow(gadd, n) if gadd is not None else 0.0)
                    a2 = _row(gax, n).numpy() if gax is not None else self._A(h, g2)
                    r2 = b - a2
                    if r2 @ r2 < r0 @ r0:
                        start = g2
                try:
                    x, its = O.cg(lambda v: self._A(h, v), b, x0=start, rel_tol=rel_tol, max_iter=max_iter)
                except O.OracleCgFailure as exc:
                    if self.fail is None:
                        self.fail = (n, exc)
                    counters += torch.tensor([1, exc.iterations, 0, 0, 0])
                    break
                counters += torch.tensor([1, its, its + 2, 0, 0])
                ax_row = self._A(h, x)
                prev = (s, b, b - ax_row)
                if ax is not None:
                    _row(ax, n // out_div).copy_(torch.from_numpy(ax_row))
                y = x
                if gadd is not None:
                    y = grow(gadd, n) + y
                if keep is not None:
                    _row(keep, n // out_div).copy_(torch.from_numpy(y))
                if sub is not None:
                    y = y - _row(sub, n).numpy()
                if out is not None:
                    _row(out, n // out_div).copy_(torch.from_numpy(y))
                if norms is not None:
                    norms[n // out_div] = float(y @ y)

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
    """Minimal Discretization stand-in used through MgritHierarchy(_disc_factory=...)."""

    def __init__(self, spec, cg_opts, engine=None):
        self.spec = spec
        self.cg_opts = cg_opts
        self.engine = engine or CpuEngine(spec.grid, spec.beta, spec.gamma, spec.kx, spec.ky)
        self.device = torch.device("cpu")
        self.counters = torch.zeros(5, dtype=torch.int64)
        self.ndof = spec.grid.ndof

    def device_loads(self, points):
        from paper_1805_06688_b200.engine import gauss_tau
        from paper_1805_06688_b200.sources import SeparableP1Source

        src = self.spec.source
        if isinstance(src, SeparableP1Source) and src.grid == self.spec.grid:  # F_n = tau_n M g (stepper.py)
            if src.kind == "zero":
                return DeviceLoads(None, 0, None)
            mg = torch.from_numpy(self.engine.ops.mass(np.asarray(src.nodal, dtype=float)))
            return DeviceLoads(mg, 0, torch.from_numpy(gauss_tau(points, src.time_factor)))
        prob = O.Problem(O.Grid(self.spec.grid.mx, self.spec.grid.my), points, self.spec.kx, self.spec.ky,
                         self.spec.beta, self.spec.gamma, self.spec.source, self.spec.initial)
        st = O.Stepper(prob)
        F = np.zeros((points.size, self.ndof))
        for n in range(1, points.size):
            F[n] = st.load(n)
        return DeviceLoads(torch.from_numpy(F), self.ndof, None)


def cpu_disc_factory(spec, cg_opts, engine):
    return CpuDisc(spec, cg_opts, engine)
