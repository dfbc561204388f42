"""Time-slab decomposition of the MGRIT hierarchy over ranks.

One process per GPU.  Rank p owns the contiguous block of fine time points
(T_p, T_{p+1}] (rank 0 also owns point 0).  The block boundaries are multiples
of m^(L-1) fine points (L = number of levels), so on every level the boundary
falls on a C-point and every interval (chain) of every level lies inside one
rank: F-relaxation, C-relaxation, restriction and correction are rank-local.
The only exchanges are

* the left C-point U[lo] of the slab, sent by its owner before each
  F-relaxation (one ndof FP64 vector per slab boundary, NCCL send/recv);
* the coarsest level, solved as a rank-ordered pipeline (each rank receives
  the value at its left boundary, forward-substitutes its points, sends on);
* per-point squared residual norms and the solve counters, combined with an
  all-reduce SUM over disjoint entries (exact), then summed on the host in
  global time-index order -- traces are bitwise identical for any rank count
  because chain results never depend on the partition (csrc/rm_device.cuh).

``torch.distributed`` is the plumbing (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["SlabPlan", "Comm", "make_plan"]


@dataclass(frozen=True)
class SlabPlan:
    """Owned level-l point ranges (lo, hi] for every rank and level."""

    world: int
    rank: int
    ranges: tuple  # ranges[l][p] = (lo, hi) in level-l indices

    def own(self, l: int) -> tuple[int, int]:
        return self.ranges[l][self.rank]

    def owner(self, l: int, n: int) -> int:
        """Rank owning level-l point n (point 0 belongs to rank 0)."""
        if n == 0:
            return 0
        for p, (lo, hi) in enumerate(self.ranges[l]):
            if lo < n <= hi:
                return p
        raise ValueError(f"point {n} of level {l} has no owner")

    def left_source(self, l: int) -> int | None:
        """Rank that holds U[lo] of this rank's slab on level l (None: own or nothing to do)."""
        lo, hi = self.own(l)
        if hi <= lo or lo == 0:
            return None
        return self.owner(l, lo)

    def right_targets(self, l: int) -> list[int]:
        """Ranks whose left boundary is this rank's last point on level l."""
        lo, hi = self.own(l)
        if hi <= lo:
            return []
        return [p for p, (a, b) in enumerate(self.ranges[l]) if b > a and a == hi]


def make_plan(n_levels_points: list[int], m: int, world: int, rank: int) -> SlabPlan:
    """Balanced partition of the fine points aligned to m^(L-1) (m^(L-2) chains at level 0)."""
    L = len(n_levels_points)
    N = n_levels_points[0]
    align = m ** max(L - 1, 0) if L > 1 else 1
    blocks = N // align
    if world > blocks:
        raise ValueError(f"{world} ranks but only {blocks} aligned time blocks of {align} steps "
                         f"(N={N}, m={m}, {L} levels); use fewer ranks or fewer levels")
    bounds = [align * ((blocks * p) // world) for p in range(world + 1)]
    ranges = []
    for l in range(L):
        scale = m**l
        ranges.append(tuple((bounds[p] // scale, bounds[p + 1] // scale) for p in range(world)))
    return SlabPlan(world, rank, tuple(ranges))


class Comm:
    """Thin wrapper over torch.distributed for the slab exchanges."""

    def __init__(self, plan: SlabPlan, group=None):
        self.plan = plan
        self.group = group

    @property
    def world(self) -> int:
        return self.plan.world

    @property
    def rank(self) -> int:
        return self.plan.rank

    def halo_left(self, U: torch.Tensor, l: int) -> None:
        """Refresh U[lo] (left boundary C-point of this rank's slab) from its owner."""
        import torch.distributed as dist

        ops = []
        src = self.plan.left_source(l)
        lo, hi = self.plan.own(l)
        if src is not None and src != self.rank:
            ops.append(dist.P2POp(dist.irecv, U[lo], src, group=self.group))
        for dst in self.plan.right_targets(l):
            if dst != self.rank:
                ops.append(dist.P2POp(dist.isend, U[hi], dst, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def recv_row(self, row: torch.Tensor, src: int) -> None:
        import torch.distributed as dist

        dist.recv(row, src, group=self.group)

    def send_row(self, row: torch.Tensor, dst: int) -> None:
        import torch.distributed as dist

        dist.send(row, dst, group=self.group)

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place SUM all-reduce (exact for disjoint contributions and for integers)."""
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t
