"""Host-side properties of the operator descriptions (reference tests/test_assembly.py: generator layout and validation,
mass generators, the single-DOF mass value, the sign of the stiffness scale, symmetric / non-symmetric blocks, SPD of the
combined stiffness and of the implicit side, the dense cap, sign validation).  Dense instantiation is host numpy; the
device applies are checked against it in tests/test_gpu_assembly.py."""

import numpy as np
import pytest

from paper_1805_06688_b200 import assembly
from paper_1805_06688_b200.assembly import (ToeplitzGenerator, combined_step_operator, mass_generators, mass_operator,
                                            stiffness_generators, stiffness_operator_x, stiffness_operator_y)
from paper_1805_06688_b200.mesh import SpatialGrid


def test_toeplitz_generator_layout_and_validation():
    gen = ToeplitzGenerator([1.0, 2.0, 3.0], [1.0, 9.0, 8.0])
    assert gen.dense == pytest.approx(np.array([[1.0, 9.0, 8.0], [2.0, 1.0, 9.0], [3.0, 2.0, 1.0]]))
    with pytest.raises(ValueError):
        ToeplitzGenerator([1.0, 2.0], [3.0, 4.0])  # corner mismatch
    with pytest.raises(ValueError):
        ToeplitzGenerator([1.0, 2.0], [1.0])  # length mismatch


def test_mass_generators_and_single_dof_value():
    grid = SpatialGrid(4, 4)
    m1, m2, scale = mass_generators(grid)
    assert scale == pytest.approx(grid.hx * grid.hy / 12.0)
    assert m1.first_col == pytest.approx([6.0, 1.0, 0.0])
    assert m2.first_row == pytest.approx([1.0, 1.0, 0.0])
    assert m2.first_col == pytest.approx([1.0, 0.0, 0.0])
    one = SpatialGrid(2, 2)  # one interior hat function: integral of phi^2 over its six triangles
    assert mass_operator(one).dense().item() == pytest.approx(one.hx * one.hy / 2.0)
    dense = mass_operator(SpatialGrid(5, 4)).dense()
    assert np.allclose(dense, dense.T) and np.linalg.eigvalsh(dense).min() > 0


@pytest.mark.parametrize("rho", [0.55, 0.75, 0.95])
def test_a1_symmetric_a2_not(rho):
    a1, a2 = stiffness_generators(6, rho)
    assert np.allclose(a1.dense, a1.dense.T)
    assert not np.allclose(a2.dense, a2.dense.T)


@pytest.mark.parametrize("beta,gamma", [(0.6, 0.9), (0.75, 0.75), (0.95, 0.55)])
def test_combined_stiffness_spd(beta, gamma):
    grid = SpatialGrid(5, 4)
    K = 2.0 * stiffness_operator_x(grid, beta).dense() + 0.5 * stiffness_operator_y(grid, gamma).dense()
    assert np.allclose(K, K.T, atol=1e-12 * np.abs(K).max())
    assert np.linalg.eigvalsh(0.5 * (K + K.T)).min() > 0


def test_scale_sign_cap_and_bad_sign():
    grid = SpatialGrid(4, 4)
    assert stiffness_operator_x(grid, 0.8).scale < 0  # 1 / (2 cos(rho pi)) is negative on (1/2, 1)
    with pytest.raises(ValueError, match="cap"):
        mass_operator(SpatialGrid(100, 100)).dense(cap=64)
    with pytest.raises(ValueError):
        combined_step_operator(mass_operator(grid), stiffness_operator_x(grid, 0.8), stiffness_operator_y(grid, 0.8),
                               1.0, 1.0, 0.1, 2)
    op = mass_operator(grid)
    assert assembly.dense_instantiation(op) == pytest.approx(op.dense())


def test_implicit_side_spd_and_dense_combination():
    grid = SpatialGrid(5, 5)
    mass, sx, sy = mass_operator(grid), stiffness_operator_x(grid, 0.9), stiffness_operator_y(grid, 0.9)
    dense = combined_step_operator(mass, sx, sy, 3.0, 7.5, 0.25, +1).dense()
    assert np.linalg.eigvalsh(0.5 * (dense + dense.T)).min() > 0
    for sign in (+1, -1):
        op = combined_step_operator(mass, sx, sy, 2.0, 0.5, 0.125, sign)
        assert op.dense() == pytest.approx(mass.dense() + sign * 0.0625 * (2.0 * sx.dense() + 0.5 * sy.dense()))
