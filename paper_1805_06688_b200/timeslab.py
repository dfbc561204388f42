"""Time-slab decomposition of the MGRIT hierarchy over ranks.

One process per GPU.  The hierarchy's levels 0 .. D-1 are DISTRIBUTED: rank p owns the contiguous block of
level-l points (lo, hi] (rank 0 also point 0), and stores only the rows lo .. hi of every level array (row lo
is the left boundary C-point: its own point on rank 0, a halo copy elsewhere).  Block boundaries are multiples
of m^D fine points, so on every distributed level the boundary falls on a C-point and every interval (chain)
lies inside one rank: F-relaxation, C-relaxation, restriction and correction are rank-local.  The coarser
levels D .. L-1 (fewer intervals than ranks) are GATHERED: rank 0 holds them in full and runs that part of
the V-cycle alone, with the single-rank code.  D is the deepest split with at least one level-(D-1) interval
per rank, so rank counts up to N/m work (config 3 at 8 ranks: D = 2, levels 16384 and 1024 distributed,
64 and 4 on rank 0).  The exchanges are

* the left C-point U[lo] of each distributed slab before every F-relaxation (one ndof FP64 vector per slab
  boundary, send/recv -- NCCL on GPUs);
* the restriction to level D: each rank's coarse rows go to rank 0 (gather); the coarse corrections come back
  (scatter);
* per-point squared residual norms and the solve counters, combined with an all-reduce SUM over disjoint
  entries (exact), then summed on the host in global time-index order -- traces are bitwise identical for any
  rank count because chain results never depend on the partition (csrc/rm_device.cuh);
* the result: each rank's rows go to rank 0 (gather), only when a host array is requested.

``torch.distributed`` is the plumbing (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

__all__ = ["SlabPlan", "Comm", "make_plan", "slab_bytes"]


@dataclass(frozen=True)
class SlabPlan:
    """Owned level-l point ranges (lo, hi] for every rank of the distributed levels l < n_dist."""

    world: int
    rank: int
    n_dist: int    # levels 0 .. n_dist-1 are distributed; n_dist .. L-1 live on rank 0
    ranges: tuple  # ranges[l][p] = (lo, hi) in level-l indices, l < n_dist
    n_points: tuple  # N_l of every level

    def own(self, l: int) -> tuple[int, int]:
        if l < self.n_dist:
            return self.ranges[l][self.rank]
        return (0, self.n_points[l]) if self.rank == 0 else (0, 0)

    def distributed(self, l: int) -> bool:
        return l < self.n_dist

    def owner(self, l: int, n: int) -> int:
        """Rank owning level-l point n (point 0 and every gathered level belong to rank 0)."""
        if n == 0 or l >= self.n_dist:
            return 0
        for p, (lo, hi) in enumerate(self.ranges[l]):
            if lo < n <= hi:
                return p
        raise ValueError(f"point {n} of level {l} has no owner")

    def left_source(self, l: int) -> int | None:
        """Rank that holds U[lo] of this rank's slab on level l (None: own or nothing to do)."""
        lo, hi = self.own(l)
        if hi <= lo or lo == 0 or l >= self.n_dist:
            return None
        return self.owner(l, lo)

    def right_targets(self, l: int) -> list[int]:
        """Ranks whose left boundary is this rank's last point on level l."""
        lo, hi = self.own(l)
        if hi <= lo or l >= self.n_dist:
            return []
        return [p for p, (a, b) in enumerate(self.ranges[l]) if b > a and a == hi]


def make_plan(n_levels_points: list[int], m: int, world: int, rank: int) -> SlabPlan:
    """Distribute the deepest feasible prefix of the hierarchy: n_dist = D <= L-1 levels with at least one
    level-(D-1) interval per rank (blocks of m^D fine steps, balanced); a single level is not split."""
    L = len(n_levels_points)
    N = n_levels_points[0]
    if world == 1 or L == 1:
        return SlabPlan(world, rank, L if world == 1 else 0,
                        tuple(((0, n),) for n in n_levels_points) if world == 1 else (), tuple(n_levels_points))
    D = 0
    for d in range(1, L):
        if N % m**d == 0 and N // m**d >= world:
            D = d
    if D == 0:
        raise ValueError(f"{world} ranks but only {N // m} intervals of {m} steps on the fine level "
                         f"(N={N}); use at most {N // m} ranks")
    align = m**D
    blocks = N // align
    bounds = [align * ((blocks * p) // world) for p in range(world + 1)]
    ranges = tuple(tuple((bounds[p] // m**l, bounds[p + 1] // m**l) for p in range(world)) for l in range(D))
    return SlabPlan(world, rank, D, ranges, tuple(n_levels_points))


def slab_bytes(plan: SlabPlan, ndof: int, compressed_g: bool = True, device_bytes: float = 180e9) -> int:
    """Device bytes of this rank's level arrays as mgrit.MgritHierarchy allocates them: on level 0 the slab rows
    of U, of G (one row and two vectors when G is compressed, mgrit.py) and -- when they take at most a quarter
    of the device (mgrit._apply_reuse_fits) -- the stored A x rows (and A G rows of an uncompressed G); G and U
    rows on every coarser level; the kept C-point values of the residual sweep."""
    total = 0
    row = ndof * 8
    for l, n in enumerate(plan.n_points):
        lo, hi = plan.own(l)
        active = l < plan.n_dist or plan.rank == 0
        rows = hi - lo + 1 if active else 0
        if l == 0:
            reuse = 2 * rows * row <= 0.25 * device_bytes
            g_rows = 3 if compressed_g else rows * (2 if reuse else 1)
            total += (rows * (2 if reuse else 1) + g_rows) * row
        else:
            total += 2 * rows * row
    lo, hi = plan.own(0)
    m = plan.n_points[0] // plan.n_points[1] if len(plan.n_points) > 1 else 1
    total += (hi // m - lo // m) * row  # kept C-point values (mgrit.solve, reuse of the residual sweep)
    return total


class Comm:
    """Thin wrapper over torch.distributed for the slab exchanges (rows are device or host tensors)."""

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
        """Refresh local row 0 (= level point lo, the left boundary C-point) from its owner and send the own last
        row to the right neighbour.  ``U`` is the level's slab-local array (row i = point lo + i)."""
        import torch.distributed as dist

        ops = []
        src = self.plan.left_source(l)
        lo, hi = self.plan.own(l)
        if src is not None and src != self.rank:
            ops.append(dist.P2POp(dist.irecv, U[0], src, group=self.group))
        for dst in self.plan.right_targets(l):
            if dst != self.rank:
                ops.append(dist.P2POp(dist.isend, U[hi - lo], dst, group=self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def gather_rows(self, full: torch.Tensor | None, mine: torch.Tensor, first: int, l: int) -> None:
        """Rank 0: full[first_p .. first_p + rows_p) <- rank p's ``mine`` (rows of level l + 1 owned by p);
        other ranks send theirs.  Row blocks are the ranks' coarse C-point rows (k0 .. k1), in rank order."""
        import torch.distributed as dist

        if self.rank == 0:
            ops = []
            for p in range(1, self.world):
                k0, k1 = self.coarse_rows(l, p)
                if k1 >= k0:
                    ops.append(dist.P2POp(dist.irecv, full[k0:k1 + 1], p, group=self.group))
            if mine.shape[0]:
                full[first:first + mine.shape[0]].copy_(mine)
            for w in dist.batch_isend_irecv(ops) if ops else []:
                w.wait()
        elif mine.shape[0]:
            dist.send(mine.contiguous(), 0, group=self.group)

    def scatter_rows(self, full: torch.Tensor | None, mine: torch.Tensor, first: int, l: int) -> None:
        """Inverse of gather_rows: rank p's ``mine`` <- rank 0's full[k0_p .. k1_p]."""
        import torch.distributed as dist

        if self.rank == 0:
            ops = []
            for p in range(1, self.world):
                k0, k1 = self.coarse_rows(l, p)
                if k1 >= k0:
                    ops.append(dist.P2POp(dist.isend, full[k0:k1 + 1].contiguous(), p, group=self.group))
            if mine.shape[0]:
                mine.copy_(full[first:first + mine.shape[0]])
            for w in dist.batch_isend_irecv(ops) if ops else []:
                w.wait()
        elif mine.shape[0]:
            buf = torch.empty_like(mine)
            dist.recv(buf, 0, group=self.group)
            mine.copy_(buf)

    def coarse_rows(self, l: int, p: int) -> tuple[int, int]:
        """Level-(l+1) rows that rank p computes by restriction from level l: its own C-points k (k m in (lo, hi])."""
        lo, hi = self.plan.ranges[l][p]
        m = self.plan.n_points[l] // self.plan.n_points[l + 1]
        return lo // m + 1, hi // m

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place SUM all-reduce (exact for disjoint contributions and for integers)."""
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def send(self, t: torch.Tensor, dst: int) -> None:
        import torch.distributed as dist

        dist.send(t.contiguous(), dst, group=self.group)

    def recv(self, t: torch.Tensor, src: int) -> None:
        import torch.distributed as dist

        dist.recv(t, src, group=self.group)
