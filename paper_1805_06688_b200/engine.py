"""Device engine: one ``rm_grid`` context plus typed wrappers of the C ABI.

Torch supplies device memory and the stream (plumbing only); every FLOP on
the path is done by the kernels in ``csrc/`` behind include/riesz_mgrit_b200.h.
There is no CPU fallback: constructing an Engine without a CUDA device, or
without the shared library, raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .krylov import CgFailure

_NVTX = os.environ.get("RM_NVTX") == "1"  # name every sweep launch for ncu --nvtx-include

__all__ = ["Engine", "require_cuda", "generators_for"]

_CG_MESSAGES = {
    1: "CG breakdown: p'Ap <= 0 or non-finite",
    2: "non-finite residual",
    3: "CG did not converge within the iteration budget",
}


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy through page-locked memory (torch's caching host allocator: repeated
    results of the same size reuse the pinned block once the previous array is released)."""
    if t.device.type != "cuda":
        return t.numpy()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)
    return host.numpy()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("riesz_mgrit_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def _ptr(t, row: int = 0) -> int | None:
    """Device address of a float64 CUDA tensor; ``(tensor, k)`` addresses row k (k may be negative)."""
    if t is None:
        return None
    off = 0
    if isinstance(t, tuple):
        t, off = t
    if t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError("device arrays must be float64 CUDA tensors")
    return t.data_ptr() + 8 * off * row


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass(frozen=True)
class Generators:
    """Host O(n) generators of one grid (assembly.py:172-274)."""

    t1x_col: np.ndarray
    t1x_row: np.ndarray
    t2x_col: np.ndarray
    t2x_row: np.ndarray
    t1y_col: np.ndarray
    t1y_row: np.ndarray
    t2y_col: np.ndarray
    t2y_row: np.ndarray
    sx: float
    sy: float
    mass_scale: float


def generators_for(grid, beta: float, gamma: float) -> Generators:
    from .assembly import stiffness_generators, stiffness_scale

    a1x, a2x = stiffness_generators(grid.mx, beta)
    a1y, a2y = stiffness_generators(grid.my, gamma)
    return Generators(a1x.first_col, a1x.first_row, a2x.first_col, a2x.first_row,
                      a1y.first_col, a1y.first_row, a2y.first_col, a2y.first_row,
                      stiffness_scale(grid.hx, grid.hy, beta), stiffness_scale(grid.hy, grid.hx, gamma),
                      grid.hx * grid.hy / 12.0)


class Engine:
    """Device operators of one spatial grid (nx x ny interior unknowns)."""

    def __init__(self, nx: int, ny: int, gens: Generators, kx: float, ky: float):
        self.device = require_cuda()
        self.lib = _native.lib()
        self.nx, self.ny = int(nx), int(ny)
        self.ndof = self.nx * self.ny
        self.kx, self.ky = float(kx), float(ky)
        self.gens = gens
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (gens.t1x_col, gens.t1x_row, gens.t2x_col, gens.t2x_row,
                 gens.t1y_col, gens.t1y_row, gens.t2y_col, gens.t2y_row)]
        for a, n in zip(arrs, (nx, nx, nx, nx, ny, ny, ny, ny)):
            if a.shape != (n,):
                raise ValueError("generator lengths must match the grid")
        self._keep = arrs
        handle = C.c_void_p()
        ptrs = [a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs]
        _native.check(self.lib.rm_grid_create(self.nx, self.ny, *ptrs, gens.sx, gens.sy, self.kx, self.ky,
                                              gens.mass_scale, C.byref(handle)), "rm_grid_create")
        self.handle = handle
        # bit 0/1: merged off-diagonal x/y matvec segments; bit 2: sweeps run the FFT kernel (rm_fft.cu)
        self.flags = int(self.lib.rm_grid_flags(handle))
        self.launches = 0
        self.trace = None  # list of (tag, start event, end event, counters-before) when profiling

    @property
    def fft(self) -> bool:
        """Sweeps of this grid run the FFT chain kernel (FP64 FFT applies and DSTs)."""
        return bool(self.flags & 4)

    def start_trace(self):
        self.trace = []

    def stop_trace(self):
        tr, self.trace = self.trace, None
        return tr

    @classmethod
    def for_problem(cls, grid, beta, gamma, kx, ky) -> "Engine":
        return cls(grid.nx, grid.ny, generators_for(grid, beta, gamma), kx, ky)

    _cache: dict = {}

    @classmethod
    def shared(cls, grid, beta, gamma, kx, ky) -> "Engine":
        """A process-wide engine per (grid, coefficients, device), reused by repeated public-API calls
        (the device context, generator tables and tau diagonals are built once)."""
        key = (grid.nx, grid.ny, float(grid.hx), float(grid.hy), float(beta), float(gamma), float(kx), float(ky),
               torch.cuda.current_device() if torch.cuda.is_available() else -1)
        eng = cls._cache.get(key)
        if eng is None:
            if len(cls._cache) >= 2:
                cls._cache.pop(next(iter(cls._cache)))
            eng = cls._cache[key] = cls.for_problem(grid, beta, gamma, kx, ky)
        return eng

    def ensure_tau(self) -> None:
        """Install the tau preconditioner (host O(n^3) setup, once per grid; precond.py)."""
        if getattr(self, "_tau_ready", False):
            return
        from .precond import tau_diagonals_from_generators

        dm, dk = tau_diagonals_from_generators(self.gens, self.nx, self.ny, self.kx, self.ky)
        dm = np.ascontiguousarray(dm, dtype=np.float64)
        dk = np.ascontiguousarray(dk, dtype=np.float64)
        _native.check(self.lib.rm_grid_set_tau(self.handle, dm.ctypes.data_as(C.POINTER(C.c_double)),
                                               dk.ctypes.data_as(C.POINTER(C.c_double))), "rm_grid_set_tau")
        self._tau_ready = True

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.rm_grid_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.handle = None

    # ------------------------------------------------------------------ apply
    def apply(self, which: int, V: torch.Tensor, dt: torch.Tensor | None = None, sign: int = 1) -> torch.Tensor:
        """out[b] = op V[b]; which 0 combined(dt[b], sign), 1 mass, 2 x-stiffness, 3 y-stiffness."""
        V = V.reshape(-1, self.ndof)
        if V.stride(1) != 1:
            V = V.contiguous()
        out = torch.empty((V.shape[0], self.ndof), dtype=torch.float64, device=V.device)
        _native.check(self.lib.rm_apply_batched(self.handle, which, V.shape[0], _ptr(dt), int(sign), _ptr(V),
                                                V.stride(0), _ptr(out), out.stride(0), _stream()),
                      "rm_apply_batched")
        self.launches += 1
        return out

    # ------------------------------------------------------------------ sweeps
    def sweep(self, *, nchains: int, first: int, cstride: int, clen: int, nmax: int, dt: torch.Tensor,
              counters: torch.Tensor, rel_tol: float, src: torch.Tensor | None = None, explicit: bool = True,
              x0_mode: int = 1, x0: torch.Tensor | None = None, f: torch.Tensor | None = None, f_stride: int = 0,
              fscale: torch.Tensor | None = None, gadd: torch.Tensor | None = None, sub: torch.Tensor | None = None,
              out: torch.Tensor | None = None, out_div: int = 1, norms: torch.Tensor | None = None,
              max_iter: int | None = None, group: int = 0, row: int | None = None, tag: str = "",
              precond: str = "none", guess=None, keep: torch.Tensor | None = None,
              hg: torch.Tensor | None = None, ax: torch.Tensor | None = None,
              gax: torch.Tensor | None = None, ain: torch.Tensor | None = None,
              gscale: torch.Tensor | None = None) -> None:
        """One rm_sweep_run launch; 2-D arrays are indexed by time point with row stride ``row``.

        ``gscale`` (compressed G): ``gadd`` and ``hg`` are single vectors, row n of each is gscale[n] times it.
        """
        if nchains <= 0:
            return
        row = self.ndof if row is None else row
        sw = _native.Sweep()
        sw.nchains, sw.first, sw.cstride, sw.clen, sw.nmax = nchains, first, cstride, clen, nmax
        sw.explicit_rhs = int(bool(explicit))
        sw.x0_mode = int(x0_mode)
        sw.out_div = int(out_div)
        sw.d_dt = _ptr(dt, 1)
        sw.d_src, sw.src_stride = _ptr(src, row), row
        sw.d_x0, sw.x0_stride = _ptr(x0, row), row
        sw.d_f, sw.f_stride = _ptr(f, int(f_stride)), int(f_stride)
        sw.d_fscale = _ptr(fscale, 1)
        sw.d_gadd, sw.gadd_stride = _ptr(gadd, row), row
        sw.d_sub, sw.sub_stride = _ptr(sub, row), row
        sw.d_out, sw.out_stride = _ptr(out, row), row
        sw.d_norms = _ptr(norms, 1)
        sw.d_guess, sw.guess_stride = _ptr(guess, row), row
        sw.d_keep, sw.keep_stride = _ptr(keep, row), row
        sw.d_hg, sw.hg_stride = _ptr(hg, row), row
        if gscale is not None:  # one stored vector each, scaled per row by gscale[n]
            sw.d_gadd, sw.gadd_stride = _ptr(gadd), 0
            sw.d_hg, sw.hg_stride = _ptr(hg), 0
            sw.d_gscale = _ptr(gscale, 1)
        sw.d_ax, sw.ax_stride = _ptr(ax, row), row
        sw.d_gax, sw.gax_stride = _ptr(gax, row), row
        sw.d_ain, sw.ain_stride = _ptr(ain, row), row
        sw.rel_tol = float(rel_tol)
        sw.max_iter = -1 if max_iter is None else int(max_iter)
        if counters.dtype != torch.int64 or not counters.is_cuda or counters.numel() < 5:
            raise TypeError("counters must be an int64 CUDA tensor of length 5")
        sw.d_counters = counters.data_ptr()
        sw.group = int(group)
        if precond in ("tau", "tau16", "tau64"):
            # 'tau64': tau-PCG in FP64; 'tau16': its DST stages on FP16 tensor cores (FP32 accumulation);
            # 'tau': additionally the in-iteration applies A p as split-FP16 tensor-core products
            # (every stopping decision stays on the FP64 true residual)
            self.ensure_tau()
            sw.precond = 1 if precond == "tau64" else 2
            sw.lp_matvec = 1 if precond == "tau" else 0
        elif precond != "none":
            raise ValueError(f"unknown preconditioner {precond!r}")
        if self.trace is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            before = counters.clone()
            e0.record()
        if _NVTX:
            torch.cuda.nvtx.range_push(tag or "sweep")
        _native.check(self.lib.rm_sweep_run(self.handle, C.byref(sw), _stream()), "rm_sweep_run")
        if _NVTX:
            torch.cuda.nvtx.range_pop()
        self.launches += 1
        if self.trace is not None:
            e1.record()
            self.trace.append((tag, e0, e1, before, counters.clone(), nchains))

    def precond_apply(self, V: torch.Tensor, dt: torch.Tensor, precond: str = "tau") -> torch.Tensor:
        """z[b] = P(dt[b])^-1 V[b] for the tau preconditioner (probe of the solver's preconditioner; tests)."""
        V = V.reshape(-1, self.ndof).contiguous()
        B = V.shape[0]
        out = torch.empty_like(V)
        cnt = torch.zeros(5, dtype=torch.int64, device=V.device)
        dt = dt.reshape(-1).to(torch.float64).contiguous()  # step n = 1..B uses dt[n-1]
        self.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dt, counters=cnt, rel_tol=1.0,
                   explicit=False, x0_mode=3, f=(V, -1), f_stride=self.ndof, out=(out, -1), precond=precond)
        return out

    def lp_apply_probe(self, V: torch.Tensor, dt: torch.Tensor) -> torch.Tensor:
        """(M + dt[b]/2 K) V[b] through the split-FP16 in-iteration apply (probe; tests)."""
        V = V.reshape(-1, self.ndof).contiguous()
        B = V.shape[0]
        out = torch.empty_like(V)
        cnt = torch.zeros(5, dtype=torch.int64, device=V.device)
        dt = dt.reshape(-1).to(torch.float64).contiguous()
        self.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dt, counters=cnt, rel_tol=1.0,
                   explicit=False, x0_mode=4, f=(V, -1), f_stride=self.ndof, out=(out, -1), precond="tau")
        return out

    def apply_probe(self, V: torch.Tensor, dt: torch.Tensor) -> torch.Tensor:
        """(M + dt[b]/2 K) V[b] through the chain kernel's own FP64 operator (rm_sweep x0_mode 4; the FFT
        kernel's grids; probe for tests)."""
        V = V.reshape(-1, self.ndof).contiguous()
        B = V.shape[0]
        out = torch.empty_like(V)
        cnt = torch.zeros(5, dtype=torch.int64, device=V.device)
        dt = dt.reshape(-1).to(torch.float64).contiguous()
        self.sweep(nchains=B, first=1, cstride=1, clen=1, nmax=B, dt=dt, counters=cnt, rel_tol=1.0,
                   explicit=False, x0_mode=4, f=(V, -1), f_stride=self.ndof, out=(out, -1), precond="none")
        return out

    def check_fail(self) -> None:
        """Raise CgFailure for the first failed solve since the last reset (synchronises)."""
        code, n, its, res = C.c_int(), C.c_int(), C.c_int64(), C.c_double()
        hit = _native.check(self.lib.rm_fail_info(self.handle, C.byref(code), C.byref(n), C.byref(its),
                                                  C.byref(res)), "rm_fail_info")
        if hit:
            _native.check(self.lib.rm_fail_reset(self.handle, _stream()), "rm_fail_reset")
            msg = _CG_MESSAGES.get(code.value, "CG failure")
            err = CgFailure(f"{msg} (time index {n.value}, iteration {its.value}, residual {res.value:.3e})",
                            res.value, its.value)
            err.time_index = n.value
            err.code = code.value
            raise err

    # ------------------------------------------------------------------ helpers
    def correct(self, U: torch.Tensor, Uc: torch.Tensor, m: int) -> None:
        nc = Uc.shape[0] - 1
        _native.check(self.lib.rm_correct(self.ndof, nc, m, _ptr(U), U.stride(0), _ptr(Uc), Uc.stride(0),
                                          _stream()), "rm_correct")
        self.launches += 1

    def diff_sqnorm(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
        _native.check(self.lib.rm_diff_sqnorm(a.numel(), _ptr(a), _ptr(b), _ptr(out), _stream()),
                      "rm_diff_sqnorm")
        self.launches += 1

    def pcg64_fill(self, seed: int, out: torch.Tensor, start: int = 0) -> None:
        """out[:] = draws start.. of np.random.default_rng(seed).random(), generated on the device."""
        st = np.random.default_rng(seed).bit_generator.state["state"]
        s, inc = int(st["state"]), int(st["inc"])
        mask = (1 << 64) - 1
        rows, row = out.shape
        _native.check(self.lib.rm_pcg64_uniform(s >> 64, s & mask, inc >> 64, inc & mask, int(start), rows * row,
                                                row, _ptr(out), out.stride(0), _stream()), "rm_pcg64_uniform")
        self.launches += 1


def gauss_tau(points: np.ndarray, factor, nq: int = 2) -> np.ndarray:
    """tau_n = sum_q (dt/2) w_q s(t_q) for n = 1..N (index 0 unused; stepper.py:129-140)."""
    xg, wg = np.polynomial.legendre.leggauss(nq)
    tau = np.zeros(points.size)
    for n in range(1, points.size):
        t0, t1 = points[n - 1], points[n]
        mid, half = (t0 + t1) / 2.0, (t1 - t0) / 2.0
        acc = 0.0
        for xi, wi in zip(xg, wg):
            acc += (half * wi) * factor(mid + half * xi)
        tau[n] = acc
    return tau
