"""Multi-rank time-slab MGRIT on the CPU: gloo backend, world sizes 2 and 4.

The chain computations run in the oracle-backed CPU engine (tests/cpu_engine.py);
what is tested is the host-side distribution: slab partition, left C-point
halo exchange before every F-relaxation, coarsest-level pipeline, exact
combination of residual norms and counters, result assembly.  The distributed
trace and solution must be BITWISE equal to the single-rank run.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import REPO, manufactured
from paper_1805_06688_b200.mesh import SpatialGrid, uniform_temporal
from paper_1805_06688_b200.mgrit import MgritOptions, solve
from paper_1805_06688_b200.stepper import ProblemSpec
from paper_1805_06688_b200.timeslab import make_plan


def test_plan_aligned_partition():
    # cfg2 structure: 4096 / 512 / 64 / 8 points, m = 8 -> blocks of 512 fine steps
    plan = make_plan([4096, 512, 64, 8], 8, 8, 3)
    assert plan.own(0) == (1536, 2048)
    assert plan.own(1) == (192, 256)
    assert plan.own(2) == (24, 32)
    assert plan.own(3) == (3, 4)
    assert plan.left_source(0) == 2 and plan.right_targets(0) == [4]
    assert plan.owner(3, 0) == 0 and plan.owner(3, 8) == 7
    with pytest.raises(ValueError, match="aligned"):
        make_plan([4096, 512, 64, 8], 8, 16, 0)
    # uneven split: 3 ranks over 8 blocks
    p3 = [make_plan([4096, 512, 64, 8], 8, 3, r).own(0) for r in range(3)]
    assert p3[0][0] == 0 and p3[-1][1] == 4096
    assert all(a[1] == b[0] for a, b in zip(p3, p3[1:]))
    assert all((hi - lo) % 512 == 0 for lo, hi in p3)


def _spec():
    c = manufactured()
    return ProblemSpec(SpatialGrid(6, 6), uniform_temporal(1.0, 64), c["kx"], c["ky"], c["beta"], c["gamma"],
                       c["source"], c["initial"])


OPTS = {
    "multi": dict(m=4, halt_tol=1e-10, cg_rel_tol=1e-12, cg_preconditioner="none"),
    "two": dict(m=4, max_levels=2, halt_tol=1e-10, cg_rel_tol=1e-12, cg_preconditioner="none"),
    "noskip_f": dict(m=2, halt_tol=1e-10, cg_rel_tol=1e-12, relaxation="f", skip_first_down=False,
                     cg_preconditioner="none"),
}


def _run(tag, distributed):
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from cpu_engine import cpu_disc_factory

    U, tr = solve(_spec(), MgritOptions(**OPTS[tag]), disc_factory=cpu_disc_factory, distributed=distributed)
    return U, tr


def _worker(rank, world, port, tags, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for tag in tags:
            U, tr = _run(tag, True)
            q.put((tag, rank, U, tr.residual_norms, tr.spatial_solves, tr.cg_iterations))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,tags", [(2, ("multi", "two", "noskip_f")), (4, ("multi",))])
def test_distributed_trace_bitwise_equal(world, tags):
    single = {tag: _run(tag, False) for tag in tags}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tags, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=900) for _ in range(world * len(tags))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for tag, rank, U, res, solves, cgits in results:
        U1, tr1 = single[tag]
        assert res == tr1.residual_norms, (tag, rank)
        assert solves == tr1.spatial_solves, (tag, rank)
        assert cgits == tr1.cg_iterations, (tag, rank)
        assert np.array_equal(U, U1), (tag, rank)


OPTS["noskip_fcf"] = dict(m=4, halt_tol=1e-10, cg_rel_tol=1e-12, skip_first_down=False, cg_preconditioner="none")


@pytest.mark.parametrize("tag", ["multi", "two", "noskip_f", "noskip_fcf"])
def test_single_rank_driver_matches_oracle(tag):
    """The host driver's work elision (residual F-relaxation done in place, the C-relaxation taken from
    the values the residual sweep kept) reproduces the reference's trace: same residual norms, spatial
    solve and CG iteration counts as the oracle's straight restatement of mgrit.py:200-322."""
    from oracle import riesz_oracle as O

    U, tr = _run(tag, False)
    spec = _spec()
    prob = O.Problem(O.Grid(spec.grid.mx, spec.grid.my), spec.tmesh.points, spec.kx, spec.ky, spec.beta, spec.gamma,
                     spec.source, spec.initial)
    o = {k: v for k, v in OPTS[tag].items() if k != "cg_preconditioner"}
    R, rtr = O.mgrit_solve(prob, O.Options(**o))
    assert tr.iterations == rtr.iterations
    assert tr.spatial_solves == rtr.spatial_solves
    assert tr.cg_iterations == rtr.cg_iterations
    np.testing.assert_allclose(tr.residual_norms, rtr.residual_norms, rtol=1e-9)
    np.testing.assert_allclose(U, R, rtol=0, atol=1e-13 * np.abs(R).max())
