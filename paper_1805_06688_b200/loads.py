"""Source load vectors (mirrors riesz_mgrit/quadrature.py + Discretization.load_vector).

Host-side setup, not on the hot path.  Two routes:

* ``SeparableP1Source`` (the BASELINE inputs): F_n = tau_n * M_h g exactly,
  with ``tau_n = sum_q (dt/2) w_q s(t_q)`` -- one device mass apply for the
  whole run plus one scalar per time step;
* any other callable: the reference quadrature (criss-cross triangles, edge
  midpoint rule subdivided ``refine`` times or the 7-point Radon rule, times
  ``time_quad_points``-point Gauss in time; quadrature.py:18-131,
  stepper.py:129-140) evaluated on the host.
"""

from __future__ import annotations

import numpy as np

from .mesh import SpatialGrid

__all__ = ["triangle_rule", "HatQuadrature"]

_R7 = (0.059715871789770, 0.470142064105115, 0.132394152788506,
       0.797426985353087, 0.101286507323456, 0.125939180544827)


def triangle_rule(rule: str = "midpoint", refine: int = 0):
    """Barycentric points (q, 3) and weights summing to one (quadrature.py:23-67)."""
    if rule == "midpoint":
        pts = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])
        w = np.full(3, 1.0 / 3.0)
    elif rule == "radon7":
        a1, b1, w1, a2, b2, w2 = _R7
        pts = np.array([[1 / 3, 1 / 3, 1 / 3], [a1, b1, b1], [b1, a1, b1], [b1, b1, a1],
                        [a2, b2, b2], [b2, a2, b2], [b2, b2, a2]])
        w = np.array([9 / 40, w1, w1, w1, w2, w2, w2])
    else:
        raise ValueError(f"unknown rule {rule!r}")
    tris = [np.eye(3)]
    for _ in range(refine):
        nxt = []
        for a, b, c in tris:
            ab, bc, ca = (a + b) / 2, (b + c) / 2, (c + a) / 2
            nxt.extend([np.array([a, ab, ca]), np.array([ab, b, bc]), np.array([ca, bc, c]), np.array([ab, bc, ca])])
        tris = nxt
    return np.vstack([pts @ t for t in tris]), np.concatenate([w / len(tris)] * len(tris))


class HatQuadrature:
    """Integrals of f * phi_j over supp(phi_j) from point values of f."""

    def __init__(self, grid: SpatialGrid, rule: str = "midpoint", refine: int = 1):
        self.grid = grid
        bary, w = triangle_rule(rule, refine)
        mx, my = grid.mx, grid.my
        ii, jj = np.meshgrid(np.arange(mx), np.arange(my))
        ii, jj = ii.ravel(), jj.ravel()
        corners = []  # (node i, node j) of the three vertices, lower then upper triangles
        for di, dj in ((0, 0), (1, 0), (1, 1)):
            corners.append((ii + di, jj + dj))
        lower = corners
        upper = [(ii, jj), (ii + 1, jj + 1), (ii, jj + 1)]
        tri_i = np.vstack([np.stack([c[0] for c in lower], 1), np.stack([c[0] for c in upper], 1)])
        tri_j = np.vstack([np.stack([c[1] for c in lower], 1), np.stack([c[1] for c in upper], 1)])
        x = grid.a + grid.hx * tri_i
        y = grid.c + grid.hy * tri_j
        self.px = (x @ bary.T).ravel()
        self.py = (y @ bary.T).ravel()
        interior = (tri_i > 0) & (tri_i < mx) & (tri_j > 0) & (tri_j < my)
        dof = np.where(interior, (tri_j - 1) * (mx - 1) + (tri_i - 1), -1)
        q = bary.shape[0]
        area = grid.hx * grid.hy / 2.0
        rows, cols, vals = [], [], []
        pid = np.arange(tri_i.shape[0] * q).reshape(-1, q)
        for v in range(3):
            keep = dof[:, v] >= 0
            for k in range(q):
                rows.append(dof[keep, v])
                cols.append(pid[keep, k])
                vals.append(np.full(int(keep.sum()), area * w[k] * bary[k, v]))
        from scipy.sparse import csr_matrix

        self.W = csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                            shape=(grid.ndof, tri_i.shape[0] * q))

    def integrate_against_hats(self, fvals: np.ndarray) -> np.ndarray:
        return self.W @ fvals
