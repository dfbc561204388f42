"""Conjugate Gradient on the device (mirrors riesz_mgrit/krylov.py).

``cg_solve`` keeps the reference signature and stopping rule (krylov.py:32-92):
unpreconditioned CG, convergence when ||r|| <= rel_tol*||rhs|| (absolute
rel_tol when rhs = 0), acceptance re-checked on the true residual with a
restart on drift, ``CgFailure`` on breakdown / non-finite values / budget.
The solve itself runs in the chain kernel (csrc/rm_kernels.cu); the operator
must be this package's implicit-side ``CombinedStepOperator`` (the only SPD
operator on the path).  Arbitrary Python callables are not accepted: there is
no CPU fallback.  Extension: ``rhs`` may be a batch ``[B, ndof]``, solved
concurrently.
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

    if not isinstance(op, CombinedStepOperator) or op.sign != +1:
        raise TypeError("cg_solve runs on the device and needs the implicit-side CombinedStepOperator (sign=+1)")
    return op._device_solve(rhs, x0, opts or CgOptions())
