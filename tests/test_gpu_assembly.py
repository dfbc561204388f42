"""Device applies of the block-Toeplitz operators against their host dense instantiation (reference
tests/test_assembly.py:95-160: apply == dense @ v on a rectangular grid, the y-direction apply against the permuted
y-fastest product, the combined step operator for both signs)."""

import numpy as np
import pytest

from paper_1805_06688_b200.assembly import (combined_step_operator, mass_operator, permutation_to_column_major,
                                            stiffness_operator_x, stiffness_operator_y)
from paper_1805_06688_b200.mesh import SpatialGrid

pytestmark = pytest.mark.gpu


def host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


@pytest.mark.parametrize("shape", [(7, 5), (5, 9), (16, 16)])
def test_apply_matches_dense(shape):
    grid = SpatialGrid(*shape)
    rng = np.random.default_rng(0)
    for op in (mass_operator(grid), stiffness_operator_x(grid, 0.8), stiffness_operator_y(grid, 0.65)):
        v = rng.standard_normal(grid.ndof)
        assert host(op.apply(v)) == pytest.approx(op.dense() @ v, abs=1e-12)
        V = rng.standard_normal((3, grid.ndof))  # a batch
        assert host(op.apply(V)) == pytest.approx(V @ op.dense().T, abs=1e-12)


def test_y_apply_matches_permuted_product():
    grid = SpatialGrid(5, 4)
    op = stiffness_operator_y(grid, 0.75)
    T1, T2 = op.diag_block.dense, op.off_block.dense
    nx = grid.mx - 1
    up = np.eye(nx, k=1)
    B = op.scale * (np.kron(np.eye(nx), T1) + np.kron(up, T2) + np.kron(up.T, T2.T))
    P = np.eye(grid.ndof)[permutation_to_column_major(grid)]
    v = np.random.default_rng(1).standard_normal(grid.ndof)
    assert host(op.apply(v)) == pytest.approx(P.T @ B @ P @ v, abs=1e-12)


def test_combined_apply_and_dense_agree():
    grid = SpatialGrid(8, 8)
    mass, sx, sy = mass_operator(grid), stiffness_operator_x(grid, 0.8), stiffness_operator_y(grid, 0.7)
    v = np.random.default_rng(2).standard_normal(grid.ndof)
    for sign in (+1, -1):
        op = combined_step_operator(mass, sx, sy, 2.0, 0.5, 0.125, sign)
        expected = mass.dense() @ v + sign * 0.0625 * (2.0 * sx.dense() @ v + 0.5 * sy.dense() @ v)
        assert host(op.apply(v)) == pytest.approx(expected, abs=1e-12)
        assert op.dense() @ v == pytest.approx(expected, abs=1e-12)
