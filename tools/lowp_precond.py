"""Precision study for the tau preconditioner's DST stages (CPU, numpy).

PCG iteration counts to the reference tolerance (1e-12) with the DST matrices S and the stage data rounded
to a given number of mantissa bits (FP32 accumulation), against exact FP64 stages, on BASELINE config 2's
operator (127^2) for warm-started propagations at several dt:

    python tools/lowp_precond.py

Result (committed in DESIGN.md): the data tolerates bf16 (7 bits); S does not (bf16 S costs up to +7 %
iterations), a two-term bf16 split of S (~16 bits) or 10-bit S restores the FP64 counts.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_06688_b200.assembly import mass_generators, stiffness_generators, stiffness_scale  # noqa: E402
from paper_1805_06688_b200.configs import make_case  # noqa: E402
from paper_1805_06688_b200.precond import dst_matrix, tau_diagonals  # noqa: E402


def rnd(a, bits):
    if bits is None:
        return a
    a32 = a.astype(np.float32)
    if bits >= 23:
        return a32.astype(np.float64)
    i = a32.view(np.uint32).astype(np.uint64)
    drop = 23 - bits
    i = ((i + (1 << (drop - 1))) >> drop) << drop
    return i.astype(np.uint32).view(np.float32).astype(np.float64)


def make_prec(S, d, n, sbits, dbits, split):
    if sbits is None:
        def P(r):
            return (S @ ((S @ r.reshape(n, n) @ S) / d) @ S).ravel()
        return P
    terms = [rnd(S, sbits)]
    if split:
        terms.append(rnd(S - terms[0], sbits))

    def mm(B):  # sum_t S_t B with B rounded, FP32 accumulation
        Bq = rnd(B, dbits).astype(np.float32)
        return sum((T.astype(np.float32) @ Bq).astype(np.float64) for T in terms)

    def P(r):
        T = mm(r.reshape(n, n).T).T  # x-stage
        T = mm(T) / d                # y-stage, diagonal
        T = mm(T.T).T
        return mm(T).ravel()
    return P


def pcg(A, b, P, x0, tol=1e-12, maxit=500):
    x = x0.copy()
    r = b - A(x)
    z = P(r)
    p = z.copy()
    rz = r @ z
    nb = np.linalg.norm(b)
    for k in range(1, maxit):
        Ap = A(p)
        a = rz / (p @ Ap)
        x += a * p
        r -= a * Ap
        if np.linalg.norm(r) <= tol * nb:
            return k
        z = P(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit


class StepOps:
    """(M + sign dt/2 (kx Ax + ky Ay)) v on the host for the study (BTTB blocks, assembly.py:100-161 layout)."""

    def __init__(self, case):
        g = case.grid
        self.n = g.nx
        m1, m2, self.cm = mass_generators(g)
        a1x, a2x = stiffness_generators(g.mx, case.beta)
        a1y, a2y = stiffness_generators(g.my, case.gamma)
        self.mass = (m1.dense, m2.dense)
        self.sx = (case.kx * stiffness_scale(g.hx, g.hy, case.beta), a1x.dense, a2x.dense)
        self.sy = (case.ky * stiffness_scale(g.hy, g.hx, case.gamma), a1y.dense, a2y.dense)

    @staticmethod
    def _x(V, T1, T2):
        W = V @ T1.T
        W[:-1] += V[1:] @ T2.T
        W[1:] += V[:-1] @ T2
        return W

    @staticmethod
    def _y(V, T1, T2):
        W = T1 @ V
        W[:, :-1] += T2 @ V[:, 1:]
        W[:, 1:] += T2.T @ V[:, :-1]
        return W

    def step_apply(self, dt, sign, v):
        V = v.reshape(self.n, self.n)
        out = self.cm * self._x(V, *self.mass)
        out += (sign * dt / 2) * (self.sx[0] * self._x(V, *self.sx[1:]) + self.sy[0] * self._y(V, *self.sy[1:]))
        return out.ravel()


def main():
    case = make_case("cfg2", Nt=8)
    ops = StepOps(case)
    n = ops.n
    dm, dk = tau_diagonals(case.grid, case.beta, case.gamma, case.kx, case.ky)
    S = dst_matrix(n)
    v = np.random.default_rng(4).random((4, n * n))
    variants = [("fp64", None, None, False), ("S bf16, data bf16", 7, 7, False),
                ("S bf16 2-term split, data bf16", 7, 7, True), ("S 10 bit, data bf16", 10, 7, False),
                ("S fp16, data fp16", 10, 10, False)]
    for dt in (1 / 4096, 1 / 64, 1 / 8, 1 / 2):
        A = lambda x: ops.step_apply(dt, +1, x)  # noqa: E731
        d = dm + 0.5 * dt * dk
        row = []
        for name, sb, db, sp in variants:
            P = make_prec(S, d, n, sb, db, sp)
            row.append(f"{name}: {sum(pcg(A, ops.step_apply(dt, -1, x), P, x) for x in v)}")
        print(f"dt={dt:.6f}  " + "  ".join(row))


if __name__ == "__main__":
    main()
