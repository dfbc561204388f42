"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``riesz_mgrit`` read-only from /root/reference/pkg/src and writes
``tests/golden/*.npz``.  The fixtures pin the CPU oracle (``oracle/``) and the
GPU path; /root/reference is never read at test or bench time.
Inputs come from ``paper_1805_06688_b200.configs`` (the canonical recipe) and
the reference's own manufactured Example 4.1 (verify.py:28-74).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from riesz_mgrit import assembly  # noqa: E402
from riesz_mgrit.krylov import CgOptions, cg_solve  # noqa: E402
from riesz_mgrit.mesh import SpatialGrid, TemporalMesh, uniform_temporal  # noqa: E402
from riesz_mgrit.mgrit import MgritOptions, parareal_solve, solve  # noqa: E402
from riesz_mgrit.stepper import Discretization, ProblemSpec, sequential_solve, spacetime_residual  # noqa: E402
from riesz_mgrit.verify import make_problem, manufactured_case  # noqa: E402

from paper_1805_06688_b200.configs import make_case  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path) / 1e6:.2f} MB")


def ref_spec(case):
    kw = case.problem_kwargs()
    grid = SpatialGrid(case.grid.mx, case.grid.my)
    tmesh = TemporalMesh(case.tmesh.points)
    kw.update(grid=grid, tmesh=tmesh)
    return ProblemSpec(**kw)


def trace_arrays(prefix, trace):
    return {
        f"{prefix}_res": np.array(trace.residual_norms),
        f"{prefix}_solves": np.array(trace.spatial_solves),
        f"{prefix}_cgits": np.array(trace.cg_iterations),
    }


def operators():
    rng = np.random.default_rng(42)
    out = {}
    cases = [(7, 5, 0.8, 0.65, 2.0, 0.5), (4, 4, 0.8, 0.7, 2.0, 0.5), (17, 9, 0.6, 0.9, 1.0, 3.0),
             (32, 32, 0.7, 0.7, 1.0, 1.0), (128, 128, 0.6, 0.8, 1.0, 2.0)]
    for i, (mx, my, b, g, kx, ky) in enumerate(cases):
        grid = SpatialGrid(mx, my)
        mass = assembly.mass_operator(grid)
        sx = assembly.stiffness_operator_x(grid, b)
        sy = assembly.stiffness_operator_y(grid, g)
        V = rng.standard_normal((3, grid.ndof))
        out[f"c{i}_params"] = np.array([mx, my, b, g, kx, ky])
        out[f"c{i}_v"] = V
        out[f"c{i}_mass"] = np.stack([mass.apply(v) for v in V])
        out[f"c{i}_sx"] = np.stack([sx.apply(v) for v in V])
        out[f"c{i}_sy"] = np.stack([sy.apply(v) for v in V])
        dts = np.array([1e-3, 0.125, 1.0])
        out[f"c{i}_dts"] = dts
        for sign, tag in ((1, "imp"), (-1, "exp")):
            out[f"c{i}_{tag}"] = np.stack([
                assembly.combined_step_operator(mass, sx, sy, kx, ky, dt, sign).apply(v)
                for dt, v in zip(dts, V)])
        a1, a2 = assembly.stiffness_generators(mx, b)
        out[f"c{i}_a1"] = a1.first_col
        out[f"c{i}_a2col"] = a2.first_col
        out[f"c{i}_a2row"] = a2.first_row
        out[f"c{i}_sxscale"] = np.array(sx.scale)
        out[f"c{i}_syscale"] = np.array(sy.scale)
    save("operators.npz", **out)


def cg_cases():
    rng = np.random.default_rng(7)
    case = manufactured_case(0.6, 0.7, 2.0, 0.5)
    out = {}
    for i, (M, dt, warm, tol) in enumerate([(16, 0.01, False, 1e-12), (16, 1.0, True, 1e-12),
                                             (32, 1.0 / 256, True, 1e-12), (8, 0.5, False, 1e-9)]):
        spec = make_problem(case, SpatialGrid(M, M), uniform_temporal(1.0, 4))
        disc = Discretization(spec)
        op = disc.combined(dt, +1)
        b = rng.standard_normal(disc.ndof)
        x0 = rng.standard_normal(disc.ndof) if warm else None
        x, its = cg_solve(op, b, x0=x0, opts=CgOptions(rel_tol=tol))
        out[f"k{i}_params"] = np.array([M, dt, float(warm), tol])
        out[f"k{i}_b"] = b
        out[f"k{i}_x0"] = x0 if warm else np.zeros(disc.ndof)
        out[f"k{i}_x"] = x
        out[f"k{i}_its"] = np.array(its)
    save("cg.npz", **out)


def stepper_cases():
    case = manufactured_case(0.8, 0.7, 2.0, 0.5)
    spec = make_problem(case, SpatialGrid(4, 4), uniform_temporal(1.0, 8))
    disc = Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13))
    rng = np.random.default_rng(3)
    v = rng.standard_normal(disc.ndof)
    out = {
        "loads": np.stack([disc.load_vector(spec.tmesh.points[n - 1], spec.tmesh.points[n]) for n in range(1, 9)]),
        "gvecs": np.stack([disc.rhs_vector(n) for n in range(1, 9)]),
        "prop_v": v,
        "prop_out": disc.propagate(0.125, v),
        "seq": sequential_solve(spec, Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13))),
    }
    U = out["seq"].copy()
    U[3] += 1e-3
    norms, tot = spacetime_residual(spec, U, Discretization(spec, cg_opts=CgOptions(rel_tol=1e-13)))
    out["stres_norms"] = norms
    out["stres_total"] = np.array(tot)
    # a larger manufactured sequential solve for the GPU chain kernel
    spec2 = make_problem(case, SpatialGrid(16, 16), uniform_temporal(1.0, 32))
    out["seq16"] = sequential_solve(spec2, Discretization(spec2, cg_opts=CgOptions(rel_tol=1e-12)))
    save("stepper.npz", **out)


def mgrit_small():
    case = manufactured_case(0.8, 0.7, 2.0, 0.5)
    out = {}
    spec = make_problem(case, SpatialGrid(8, 8), uniform_temporal(1.0, 64))
    runs = {
        "two": MgritOptions(m=4, max_levels=2, halt_tol=1e-10, cg_rel_tol=1e-12),
        "multi": MgritOptions(m=4, halt_tol=1e-10, cg_rel_tol=1e-12),
        "noskip": MgritOptions(m=4, halt_tol=1e-10, cg_rel_tol=1e-12, skip_first_down=False),
        "frelax": MgritOptions(m=2, halt_tol=1e-10, cg_rel_tol=1e-12, relaxation="f"),
        "seed3": MgritOptions(m=8, halt_tol=1e-10, cg_rel_tol=1e-12, rng_seed=3),
    }
    for tag, opts in runs.items():
        U, tr = solve(spec, opts)
        out[f"{tag}_U"] = U
        out.update(trace_arrays(tag, tr))
    U, tr = parareal_solve(spec, MgritOptions(m=8, halt_tol=1e-10, cg_rel_tol=1e-12))
    out["parareal_U"] = U
    out.update(trace_arrays("parareal", tr))
    save("mgrit_small.npz", **out)


def cfg1():
    case = make_case("cfg1")
    spec = ref_spec(case)
    out = {}
    for tag, lv in (("two", 2), ("multi", None)):
        t = time.perf_counter()
        opts = MgritOptions(m=case.m, max_levels=lv, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, rng_seed=0)
        U, tr = solve(spec, opts)
        print(f"cfg1 {tag}: {tr.iterations} its in {time.perf_counter() - t:.1f}s")
        out[f"{tag}_U"] = U
        out.update(trace_arrays(tag, tr))
    out["seq_U"] = sequential_solve(spec, Discretization(spec, cg_opts=CgOptions(rel_tol=case.cg_rel_tol)))
    out["psi0"] = case.psi0
    out["g"] = case.g
    save("cfg1.npz", **out)


def reduced():
    out = {}
    # cfg4-style graded mesh (time-dependent propagators), reduced sizes
    case = make_case("cfg4", M=16, Nt=64)
    spec = ref_spec(case)
    for tag, lv in (("g_two", 2), ("g_multi", None)):
        opts = MgritOptions(m=case.m, max_levels=lv, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
        U, tr = solve(spec, opts)
        out[f"{tag}_U"] = U
        out.update(trace_arrays(tag, tr))
    # cfg2 at full spatial size (127^2 DOF), reduced Nt
    case = make_case("cfg2", Nt=16)
    spec = ref_spec(case)
    t = time.perf_counter()
    opts = MgritOptions(m=case.m, max_levels=None, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    U, tr = solve(spec, opts)
    print(f"cfg2/Nt16: {tr.iterations} its in {time.perf_counter() - t:.1f}s")
    out["c2_U"] = U
    out.update(trace_arrays("c2", tr))
    # cfg2 structure (multilevel m=8) on a 31^2 grid with Nt=512: 3 levels
    case = make_case("cfg2", M=32, Nt=512)
    spec = ref_spec(case)
    t = time.perf_counter()
    opts = MgritOptions(m=case.m, max_levels=None, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    U, tr = solve(spec, opts)
    print(f"cfg2/M32/Nt512: {tr.iterations} its in {time.perf_counter() - t:.1f}s")
    out["c2s_U"] = U[::8].copy()
    out.update(trace_arrays("c2s", tr))
    save("reduced.npz", **out)


def big():
    """Full spatial sizes of BASELINE configs 3 (255^2) and 4 (511^2) at reduced Nt; U stored at a few points."""
    out = {}
    runs = [("c3", "cfg3", dict(Nt=32), None, (16, 32)), ("c4", "cfg4", dict(Nt=16), None, (8, 16))]
    for tag, name, kw, lv, keep in runs:
        case = make_case(name, **kw)
        spec = ref_spec(case)
        t = time.perf_counter()
        opts = MgritOptions(m=case.m, max_levels=lv, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
        U, tr = solve(spec, opts)
        print(f"{name} {kw}: {tr.iterations} its in {time.perf_counter() - t:.1f}s")
        out[f"{tag}_keep"] = np.array(keep)
        out[f"{tag}_U"] = U[list(keep)]
        out[f"{tag}_norms"] = np.linalg.norm(U, axis=1)
        out.update(trace_arrays(tag, tr))
    save("big.npz", **out)


def big_tight():
    """Config 4 at 511^2, Nt=16 solved by the reference with inner CG tolerance 1e-14: the reference's
    own 1e-12 solves are ~2e-10 away from the converged answer at this size (operator conditioning), so
    this anchors the accuracy of the preconditioned path, which is closer to the converged answer."""
    case = make_case("cfg4", Nt=16)
    spec = ref_spec(case)
    t = time.perf_counter()
    opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=1e-14)
    U, tr = solve(spec, opts)
    print(f"cfg4 tight: {tr.iterations} its in {time.perf_counter() - t:.1f}s")
    save("big_tight.npz", c4t_keep=np.array((8, 16)), c4t_U=U[[8, 16]], c4t_norms=np.linalg.norm(U, axis=1),
         **trace_arrays("c4t", tr))


def _sketch_matrix(ndof, k=8, seed=1234):
    """Fixed seeded projection: U @ R gives per-time-point fingerprints whose relative differences
    track the per-point relative L2 differences (used where storing all rows is too large)."""
    return np.random.default_rng(seed).standard_normal((ndof, k)) / np.sqrt(ndof)


def _run_and_store(fname, tag, case, keep, lv="case", threads_note=""):
    spec = ref_spec(case)
    t = time.perf_counter()
    opts = MgritOptions(m=case.m, max_levels=case.max_levels if lv == "case" else lv,
                        halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, rng_seed=0)
    U, tr = solve(spec, opts)
    wall = time.perf_counter() - t
    print(f"{fname} {tag}: {tr.iterations} its in {wall:.1f}s", flush=True)
    keep = np.array(sorted(set(int(k) for k in keep if 0 <= k <= case.tmesh.n_intervals)))
    out = {f"{tag}_keep": keep, f"{tag}_U": U[keep], f"{tag}_norms": np.linalg.norm(U, axis=1),
           f"{tag}_sketch": U @ _sketch_matrix(U.shape[1]), f"{tag}_wall_s": np.array(wall),
           f"{tag}_its": np.array(tr.iterations)}
    out.update(trace_arrays(tag, tr))
    save(fname, **out)


def cfg2_full():
    """BASELINE configs[1] at full size (127^2 x 4096, multilevel m=8): the workload bench.py timed in
    round 1.  ~3 h on the 8-core build container."""
    case = make_case("cfg2")
    N = case.tmesh.n_intervals
    _run_and_store("cfg2_full.npz", "c2f", case, [0, 1, 7, 8, 9, 511, 512, 2047, 2048, 2049, 4095, 4096])


def cfg2_split():
    """cfg2 grid and physics on the split-FP16 regime of the benched path: T = 1/8, Nt = 512, i.e. the
    full run's fine dt = 1/4096 and level-1 dt = 1/512 (levels 512/64/8)."""
    case = make_case("cfg2", Nt=512, T=0.125)
    _run_and_store("cfg2_split.npz", "c2p", case, [0, 1, 7, 8, 63, 64, 255, 256, 504, 511, 512])


def cfg3_split():
    """cfg3 grid and physics (255^2, m=16) at the full run's step sizes: T = 1/16, Nt = 1024, i.e. fine
    dt = 1/16384, level-1 dt = 1/1024, level-2 dt = 1/64 (levels 1024/64/4)."""
    case = make_case("cfg3", Nt=1024, T=1.0 / 16)
    _run_and_store("cfg3_split.npz", "c3p", case, [0, 1, 15, 16, 17, 255, 256, 511, 512, 1008, 1023, 1024])


def cfg4_diverge():
    """cfg4 physics (beta=0.55, gamma=0.9, graded t_n=(n/Nt)^2, m=8 multilevel) on 63^2 x 512: the reference's
    own MGRIT residual GROWS every cycle (the re-discretised Crank-Nicolson coarse propagators of the stiff
    fractional operator amplify the high modes), as it does on the GPU at the full 511^2 x 8192 size.  Four
    cycles are recorded; the reference raises MgritFailure, whose trace and iterate are stored."""
    from riesz_mgrit.mgrit import MgritFailure

    case = make_case("cfg4", M=64, Nt=512)
    spec = ref_spec(case)
    t = time.perf_counter()
    opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol, max_iters=4)
    try:
        solve(spec, opts)
        raise AssertionError("expected MgritFailure")
    except MgritFailure as exc:
        tr, U = exc.trace, exc.solution
    print(f"cfg4_diverge: {tr.iterations} its in {time.perf_counter() - t:.1f}s: {tr.residual_norms}", flush=True)
    keep = np.array([0, 1, 8, 64, 256, 511, 512])
    out = {"c4d_keep": keep, "c4d_U": U[keep], "c4d_norms": np.linalg.norm(U, axis=1),
           "c4d_sketch": U @ _sketch_matrix(U.shape[1])}
    out.update(trace_arrays("c4d", tr))
    save("cfg4_diverge.npz", **out)


def cfg4_fullnt():
    """cfg4 physics on its FULL graded time grid (Nt = 8192, t_n = (n/Nt)^2: every fine dt of the BASELINE
    run, levels 8192/1024/128/16/2) at a reduced 63^2 grid, where MGRIT converges."""
    case = make_case("cfg4", M=64)
    _run_and_store("cfg4_fullnt.npz", "c4n", case, [0, 1, 7, 8, 1024, 4095, 4096, 8184, 8191, 8192])


def cfg5_split():
    """cfg5 grid and physics (1023^2, m=16) at the full run's step sizes: T = 32/65536, Nt = 32, i.e. fine
    dt = 1/65536 and level-1 dt = 1/4096 (levels 32/2)."""
    case = make_case("cfg5", Nt=32, T=32.0 / 65536)
    _run_and_store("cfg5_split.npz", "c5p", case, [0, 1, 15, 16, 17, 31, 32])


def theory_cases():
    """Two-level bounds (reference theory.py:88-134) for cfg1, the cfg2 physics on 31^2 x 512 and the cfg4
    physics on 63^2 graded x 512 (where the reference's MGRIT diverges)."""
    from riesz_mgrit.theory import mode_spectrum, two_level_bound

    out = {}
    for tag, name, kw, m in (("t1", "cfg1", {}, 4), ("t2", "cfg2", dict(M=32, Nt=512), 8),
                             ("t4", "cfg4", dict(M=64, Nt=512), 8)):
        case = make_case(name, **kw)
        spec = ref_spec(case)
        sp = mode_spectrum(spec)
        rep = two_level_bound(sp, spec.tmesh, m)
        out[f"{tag}_sigmas"] = sp.sigmas
        out[f"{tag}_bound"] = np.array(rep.bound)
        out[f"{tag}_argmax"] = np.array(rep.argmax_mode)
        out[f"{tag}_per_mode"] = rep.per_mode
        print(tag, rep.bound, rep.argmax_mode, flush=True)
    save("theory.npz", **out)


def pcg64():
    rng = np.random.default_rng(0)
    st = rng.bit_generator.state["state"]
    first = rng.random(16)
    rng = np.random.default_rng(0)
    big = rng.random((8, 16129))
    offsets = np.array([0, 1, 15, 16129, 5 * 16129 + 17, 8 * 16129 - 1])
    save("pcg64.npz", state_hex=np.array([hex(st["state"]), hex(st["inc"])]), first=first,
         offsets=offsets, values=big.ravel()[offsets])


if __name__ == "__main__":
    which = sys.argv[1:] or ["operators", "cg", "stepper", "mgrit_small", "pcg64", "cfg1", "reduced"]
    fns = {"operators": operators, "cg": cg_cases, "stepper": stepper_cases, "mgrit_small": mgrit_small,
           "pcg64": pcg64, "cfg1": cfg1, "reduced": reduced, "big": big,
           "big_tight": big_tight, "cfg2_full": cfg2_full, "cfg2_split": cfg2_split,
           "cfg3_split": cfg3_split, "cfg4_diverge": cfg4_diverge,
           "cfg4_fullnt": cfg4_fullnt, "cfg5_split": cfg5_split,
           "theory": theory_cases}
    for w in which:
        t = time.perf_counter()
        fns[w]()
        print(f"{w}: {time.perf_counter() - t:.1f}s")
