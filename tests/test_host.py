"""CPU tests of the host side: metadata, generators, loads, the C-ABI library surface."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import REPO, manufactured
from paper_1805_06688_b200 import _native, assembly
from paper_1805_06688_b200.configs import CONFIGS, make_case
from paper_1805_06688_b200.loads import HatQuadrature
from paper_1805_06688_b200.mesh import (
    CfSplitting,
    SpatialGrid,
    TemporalMesh,
    coarsen,
    graded_temporal,
    shishkin_temporal,
    uniform_temporal,
)
from paper_1805_06688_b200.mgrit import IterationTrace, MgritOptions, convergence_factor
from paper_1805_06688_b200.sources import SeparableP1Source, p1_interpolate

HEADER = os.path.join(REPO, "include", "riesz_mgrit_b200.h")


# ----------------------------------------------------------------------------- mesh (tests/test_mesh.py)
def test_grid_basics():
    g = SpatialGrid(8, 4)
    assert g.hx == pytest.approx(1 / 8) and g.hy == pytest.approx(1 / 4) and g.ndof == 21
    x, y = SpatialGrid(4, 4).interior_nodes()
    assert x[:3] == pytest.approx([0.25, 0.5, 0.75]) and y[:3] == pytest.approx([0.25] * 3)
    for mx, my in ((1, 4), (4, 1)):
        with pytest.raises(ValueError):
            SpatialGrid(mx, my)
    with pytest.raises(ValueError):
        SpatialGrid(4, 4, a=1.0, b=0.0)


def test_temporal_meshes():
    m = uniform_temporal(2.0, 8)
    assert m.n_intervals == 8 and m.final_time == pytest.approx(2.0) and m.is_uniform()
    with pytest.raises(ValueError):
        TemporalMesh(np.array([0.0, 0.5, 0.5, 1.0]))
    with pytest.raises(ValueError):
        TemporalMesh(np.array([0.1, 0.5, 1.0]))
    with pytest.raises(ValueError):
        TemporalMesh(np.array([0.0]))
    s = shishkin_temporal(64, 2.0**-6)
    assert not s.is_uniform() and s.final_time == pytest.approx(1.0)
    with pytest.raises(ValueError, match="transition"):
        shishkin_temporal(8, 2.0**-3)
    g = graded_temporal(1.0, 16)
    assert np.array_equal(g.widths, np.diff((np.arange(17) / 16) ** 2))
    c = coarsen(s, 4)
    assert c.n_intervals == 16 and np.array_equal(c.points, s.points[::4])
    with pytest.raises(ValueError):
        coarsen(uniform_temporal(1.0, 10), 4)


def test_cf_splitting():
    sp = CfSplitting(12, 4)
    assert list(sp.c_indices) == [0, 4, 8, 12] and sp.n_coarse == 3
    assert sorted(list(sp.c_indices) + list(sp.f_indices)) == list(range(13))
    for args in ((12, 5), (12, 1)):
        with pytest.raises(ValueError):
            CfSplitting(*args)


def test_options_validation():
    for kw in (dict(m=1), dict(m=2, halt_tol=0.0), dict(m=2, relaxation="fcfc"), dict(m=2, max_iters=0)):
        with pytest.raises(ValueError):
            MgritOptions(**kw)


def test_convergence_factor():
    assert convergence_factor(IterationTrace(residual_norms=[10.0 * 0.1**k for k in range(7)])) == pytest.approx(0.1)
    with pytest.raises(ValueError):
        convergence_factor(IterationTrace(residual_norms=[1.0] * 5))


# ----------------------------------------------------------------------------- generators vs reference
@pytest.mark.parametrize("case", range(5))
def test_generators_bit_exact(golden, case):
    g = golden("operators.npz")
    mx, my, b, gm, kx, ky = g[f"c{case}_params"]
    a1, a2 = assembly.stiffness_generators(int(mx), b)
    assert np.array_equal(a1.first_col, g[f"c{case}_a1"])
    assert np.array_equal(a2.first_col, g[f"c{case}_a2col"])
    assert np.array_equal(a2.first_row, g[f"c{case}_a2row"])
    grid = SpatialGrid(int(mx), int(my))
    assert assembly.stiffness_operator_x(grid, b).scale == float(g[f"c{case}_sxscale"])
    assert assembly.stiffness_operator_y(grid, gm).scale == float(g[f"c{case}_syscale"])


def test_dense_instantiation_matches_golden_applies(golden):
    g = golden("operators.npz")
    mx, my, b, gm, kx, ky = g["c0_params"]
    grid = SpatialGrid(int(mx), int(my))
    V = g["c0_v"]
    for op, tag in ((assembly.mass_operator(grid), "mass"), (assembly.stiffness_operator_x(grid, b), "sx"),
                    (assembly.stiffness_operator_y(grid, gm), "sy")):
        assert np.abs(V @ op.dense().T - g[f"c0_{tag}"]).max() < 1e-12


def test_generator_validation():
    with pytest.raises(ValueError):
        assembly.stiffness_generators(8, 0.5)
    with pytest.raises(ValueError):
        assembly.stiffness_generators(1, 0.8)
    with pytest.raises(ValueError):
        assembly.ToeplitzGenerator([1.0, 2.0], [3.0, 4.0])
    with pytest.raises(ValueError, match="cap"):
        assembly.mass_operator(SpatialGrid(100, 100)).dense(cap=64)


# ----------------------------------------------------------------------------- loads
def test_host_quadrature_loads_match_reference(golden):
    g = golden("stepper.npz")
    c = manufactured()
    grid = SpatialGrid(4, 4)
    q = HatQuadrature(grid)
    xg, wg = np.polynomial.legendre.leggauss(2)
    pts = uniform_temporal(1.0, 8).points
    for n in range(1, 9):
        mid, half = (pts[n - 1] + pts[n]) / 2, (pts[n] - pts[n - 1]) / 2
        F = sum((half * w) * q.integrate_against_hats(c["source"](q.px, q.py, mid + half * x)) for x, w in zip(xg, wg))
        assert np.abs(F - g["loads"][n - 1]).max() <= 1e-15


def test_separable_source_load_equals_tau_mass_g():
    """For P1 nodal sources the reference quadrature load is tau_n * M_h g."""
    case = make_case("cfg2", M=12, Nt=4)
    q = HatQuadrature(case.grid)
    F = q.integrate_against_hats(case.source(q.px, q.py, 0.3))
    Mg = assembly.mass_operator(case.grid).dense() @ case.g
    assert np.abs(F - 0.3 * Mg).max() <= 1e-15 * np.abs(Mg).max() * 10


def test_p1_interpolant_reproduces_nodes_and_boundary():
    grid = SpatialGrid(6, 5)
    v = np.random.default_rng(0).standard_normal(grid.ndof)
    x, y = grid.interior_nodes()
    assert np.allclose(p1_interpolate(grid, v, x, y), v, atol=1e-15)
    assert np.all(p1_interpolate(grid, v, np.zeros(3), np.array([0.1, 0.5, 0.9])) == 0.0)
    src = SeparableP1Source(grid, v, "t")
    assert src(x, y, 2.0) == pytest.approx(2.0 * v)


def test_configs_recipe():
    for name in CONFIGS:
        c = make_case(name, M=8, Nt=16)
        assert c.psi0.shape == (c.grid.ndof,) and c.g.shape == (c.grid.ndof,)
    c1 = make_case("cfg1")
    assert c1.grid.ndof == 961 and c1.tmesh.n_intervals == 256 and c1.m == 4 and c1.max_levels == 2
    c2 = make_case("cfg2", Nt=8)
    assert c2.grid.ndof == 127 * 127
    c4 = make_case("cfg4", M=8, Nt=16)
    assert c4.tmesh.points[1] == pytest.approx(1 / 256)


# ----------------------------------------------------------------------------- C ABI surface
def header_functions():
    text = open(HEADER).read()
    return re.findall(r"RM_API\s+[\w\s\*]+?\b(rm_\w+)\s*\(", text)


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    names = header_functions()
    assert len(names) == 17
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTS)
    assert lib.rm_version().startswith(b"riesz_mgrit_b200")
    assert lib.rm_max_order() >= 128


def test_library_rejects_bad_arguments_without_gpu():
    lib = _native.lib()
    h = ctypes.c_void_p()
    z = (ctypes.c_double * 4)()
    st = lib.rm_grid_create(0, 4, z, z, z, z, z, z, z, z, 1.0, 1.0, 1.0, 1.0, 1.0, ctypes.byref(h))
    assert st == -1 and b"nx, ny" in lib.rm_last_error()
    st = lib.rm_grid_create(300, 4, z, z, z, z, z, z, z, z, 1.0, 1.0, 1.0, 1.0, 1.0, ctypes.byref(h))
    assert st == -3
    assert lib.rm_sweep_run(None, None, None) == -1
    assert lib.rm_apply_batched(None, 0, 1, None, 1, None, 0, None, 0, None) == -1


def test_sweep_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    fields = [f[0] for f in _native.Sweep._fields_]
    body = "".join(f'printf("%zu ", offsetof(rm_sweep, {f}));' for f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "riesz_mgrit_b200.h"\n'
                   f"int main(void) {{ {body} printf(\"%zu\\n\", sizeof(rm_sweep)); return 0; }}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [getattr(_native.Sweep, f).offset for f in fields] + [ctypes.sizeof(_native.Sweep)]
    assert got == want


def test_trace_payload_schema(tmp_path):
    """reporting.py:59-75 schema: keys, types, quarantined timing, factor only with >= 6 norms."""
    import json

    from paper_1805_06688_b200.mgrit import IterationTrace
    from paper_1805_06688_b200.reporting import trace_payload, write_trace

    tr = IterationTrace(residual_norms=[81.0, 9.0, 1.0, 0.1, 1e-2, 1e-3, 1e-4], spatial_solves=[10, 20, 30, 40, 50, 60, 70],
                        cg_iterations=[100, 200, 300, 400, 500, 600, 700], wall_times=[0.0] * 7, seed=0, converged=True)
    p = trace_payload(tr, {"config": "cfg1"})
    assert set(p) == {"config", "seed", "converged", "iterations", "residual_norms", "spatial_solves",
                      "cg_iterations", "timing", "convergence_factor"}
    assert p["iterations"] == 6 and p["timing"] == {"wall_times": [0.0] * 7}
    assert abs(p["convergence_factor"] - (1e-4 / 9.0) ** 0.2) < 1e-15
    short = IterationTrace(residual_norms=[1.0, 0.5], spatial_solves=[1, 2], cg_iterations=[3, 4])
    assert "convergence_factor" not in trace_payload(short, {})
    out = write_trace(tmp_path / "sub" / "trace.json", tr, {"b": 1, "a": 2})
    text = out.read_text()
    assert text.endswith("\n") and json.loads(text) == json.loads(json.dumps(p | {"config": {"b": 1, "a": 2}}))
    assert text.index('"cg_iterations"') < text.index('"config"')  # sort_keys=True


def test_preconditioner_names_and_options():
    """CgOptions / MgritOptions accept the inner-solver variants (krylov.py:12-20 plus the extensions) and
    reject anything else with ValueError, as the reference validates its options."""
    from paper_1805_06688_b200.krylov import CgOptions
    from paper_1805_06688_b200.mgrit import MgritOptions

    for name in ("tau", "tau16", "tau64", "none"):
        assert CgOptions(preconditioner=name).preconditioner == name
        assert MgritOptions(m=4, cg_preconditioner=name).cg_preconditioner == name
    with pytest.raises(ValueError):
        CgOptions(preconditioner="jacobi")
    with pytest.raises(ValueError):
        CgOptions(rel_tol=0.0)
