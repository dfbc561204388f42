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
           "big_tight": big_tight}
    for w in which:
        t = time.perf_counter()
        fns[w]()
        print(f"{w}: {time.perf_counter() - t:.1f}s")
