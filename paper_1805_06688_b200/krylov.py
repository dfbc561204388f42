"""Conjugate Gradient on the device (mirrors riesz_mgrit/krylov.py).

``cg_solve`` keeps the reference signature and stopping rule (krylov.py:32-92):
unpreconditioned CG, convergence when ||r|| <= rel_tol*||rhs|| (absolute
rel_tol when rhs = 0), acceptance re-checked on the true residual with a
restart on drift, ``CgFailure`` on breakdown / non-finite values / budget.
For this package's implicit-side ``CombinedStepOperator`` (the only SPD
operator on the hot path) the solve runs fused inside the chain kernels
(csrc/rm_kernels.cu, rm_fft.cu, rm_big.cu); ``rhs`` may then be a batch
``[B, ndof]``, solved concurrently.  Any other operator -- an object with
``apply`` or a bare callable, as krylov.py:44 accepts -- runs the same
algorithm with its vectors and reductions on the device (``rm_vec_dot`` /
``rm_vec_axpby``) and the operator called once per iteration (with a numpy
array, as the reference calls it, or with the device tensor when it sets
``accepts_device = True``).  There is no CPU fallback: without a CUDA device
both routes raise.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["CgOptions", "CgFailure", "cg_solve"]


@dataclass
class CgOptions:
    """krylov.py:12-20; ``max_iter=None`` means 10 * ndof.

    Extension: ``preconditioner`` = 'tau' (default) runs CG preconditioned by
    the optimal sine-transform approximation of the step operator
    (precond.py), its DST stages on FP16 tensor cores with FP32 accumulation
    and the in-iteration operator applies A p as split-FP16 tensor-core
    products (~2^-22 relative); 'tau16' keeps those applies in FP64; 'tau64'
    is the same preconditioner entirely in FP64; 'none' is the reference's
    unpreconditioned CG.  All stop on the reference criterion
    ||b - A x|| <= rel_tol ||b|| with the same FP64 true-residual acceptance,
    so solutions agree to the solve tolerance; only the iteration counts
    differ.
    """

    rel_tol: float = 1e-9
    max_iter: int | None = None
    record_iterations: bool = False
    preconditioner: str = "tau"

    def __post_init__(self):
        if self.rel_tol <= 0:
            raise ValueError("relative tolerance must be positive")
        if self.preconditioner not in ("tau", "tau16", "tau64", "none"):
            raise ValueError("preconditioner must be 'tau', 'tau16', 'tau64' or 'none'")


class CgFailure(RuntimeError):
    """CG stalled or broke down; carries the last residual norm (krylov.py:23-29)."""

    def __init__(self, message: str, residual_norm: float, iterations: int):
        super().__init__(message)
        self.residual_norm = residual_norm
        self.iterations = iterations


def cg_solve(op, rhs, x0=None, opts: CgOptions | None = None):
    """Solve ``op x = rhs`` on the device; returns ``(x, iterations)``.

    For a batched rhs the iteration count returned is the total over the batch.
    """
    from .assembly import CombinedStepOperator

    opts = opts or CgOptions()
    if isinstance(op, CombinedStepOperator) and op.sign == +1:
        return op._device_solve(rhs, x0, opts)
    return _generic_cg(op, rhs, x0, opts)


def _generic_cg(op, rhs, x0, opts: CgOptions):
    """krylov.py:44-92 for an arbitrary SPD operator: unpreconditioned CG, vectors resident on the device."""
    import ctypes as C

    import numpy as np
    import torch

    from . import _native
    from .engine import _ptr, _stream, require_cuda

    dev = require_cuda()
    lib = _native.lib()
    apply_op = op.apply if hasattr(op, "apply") else op
    on_device = bool(getattr(op, "accepts_device", False))
    as_torch = isinstance(rhs, torch.Tensor)
    b = (rhs.to(device=dev, dtype=torch.float64) if as_torch
         else torch.from_numpy(np.ascontiguousarray(np.asarray(rhs, dtype=float))).to(dev)).reshape(-1).contiguous()
    n = b.numel()
    max_iter = opts.max_iter if opts.max_iter is not None else 10 * n
    scal = torch.zeros(1, dtype=torch.float64, device=dev)

    def apply(v):
        if on_device:
            out = apply_op(v)
        else:
            out = apply_op(v.cpu().numpy())
        if not isinstance(out, torch.Tensor):
            out = torch.from_numpy(np.ascontiguousarray(np.asarray(out, dtype=float)))
        return out.to(device=dev, dtype=torch.float64).reshape(-1).contiguous()

    def dot(u, v):
        _native.check(lib.rm_vec_dot(n, _ptr(u), _ptr(v), _ptr(scal), _stream()), "rm_vec_dot")
        return float(scal.item())

    def axpby(alpha, u, beta, v, out):
        _native.check(lib.rm_vec_axpby(n, C.c_double(alpha), _ptr(u), C.c_double(beta), _ptr(v), _ptr(out), _stream()),
                      "rm_vec_axpby")

    def finish(x, k):
        if as_torch:
            return x.reshape(rhs.shape), k
        return x.cpu().numpy().reshape(np.shape(rhs)), k

    if x0 is None:
        x = torch.zeros_like(b)
    else:
        x = (x0.to(device=dev, dtype=torch.float64) if isinstance(x0, torch.Tensor)
             else torch.from_numpy(np.array(x0, dtype=float)).to(dev)).reshape(-1).clone()
    rhs_norm = dot(b, b) ** 0.5
    target = opts.rel_tol * rhs_norm if rhs_norm > 0 else opts.rel_tol
    r = torch.empty_like(b)
    axpby(1.0, b, -1.0, apply(x), r)
    rr = dot(r, r)
    res_norm = rr ** 0.5
    if res_norm <= target:
        return finish(x, 0)
    p = r.clone()
    for k in range(1, max_iter + 1):
        Ap = apply(p)
        pAp = dot(p, Ap)
        if not np.isfinite(pAp) or pAp <= 0:
            raise CgFailure(f"CG breakdown at iteration {k}: p'Ap = {pAp}", res_norm, k)
        alpha = rr / pAp
        axpby(1.0, x, alpha, p, x)
        axpby(1.0, r, -alpha, Ap, r)
        rr_new = dot(r, r)
        res_norm = rr_new ** 0.5
        if not np.isfinite(res_norm):
            raise CgFailure(f"non-finite residual at iteration {k}", res_norm, k)
        if res_norm <= target:
            axpby(1.0, b, -1.0, apply(x), r)  # acceptance on the true residual (krylov.py:71-83)
            rr_new = dot(r, r)
            true_res = rr_new ** 0.5
            if true_res <= max(target, 10 * res_norm):
                return finish(x, k)
            res_norm = true_res  # recurrence drifted: continue from the true residual
            if res_norm <= target:
                return finish(x, k)
            p = r.clone()
            rr = rr_new
            continue
        beta = rr_new / rr
        rr = rr_new
        axpby(1.0, r, beta, p, p)
    raise CgFailure(f"CG did not converge within {max_iter} iterations "
                    f"(residual {res_norm:.3e}, target {target:.3e})", res_norm, max_iter)
