"""Nodal (P1) source and initial-value callables.

BASELINE.json gives sources and initial data *per node*.  The reference
evaluates ``source(x, y, t)`` at quadrature points (stepper.py:129-140), so a
nodal field has to be handed over as a callable: the piecewise-linear
interpolant on the criss-cross triangulation (each cell split along its
lower-left -> upper-right diagonal, quadrature.py:85-88; boundary nodes carry 0).

``SeparableP1Source`` additionally exposes its structure, ``s(t) * g(x, y)``
with nodal ``g``.  For it the load vector is exactly ``tau_n * M_h g`` with
``tau_n = sum_q (dt/2) w_q s(t_q)`` (2-point Gauss, stepper.py:136-139): the
reference's quadrature integrates the product of two P1 functions exactly.
The device path uses that identity (one mass apply + one scalar per step)
instead of the quadrature; general callables go through the host quadrature
in :mod:`.loads`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .mesh import SpatialGrid

__all__ = ["p1_interpolate", "SeparableP1Source", "NodalInitial", "TIME_FACTORS"]


def p1_interpolate(grid: SpatialGrid, nodal: np.ndarray, x, y) -> np.ndarray:
    """Evaluate the P1 interpolant of interior nodal values at points (x, y)."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    mx, my = grid.mx, grid.my
    full = np.zeros((my + 1, mx + 1))
    full[1:my, 1:mx] = np.asarray(nodal, dtype=float).reshape(my - 1, mx - 1)
    sx = (x - grid.a) / grid.hx
    sy = (y - grid.c) / grid.hy
    i = np.clip(np.floor(sx).astype(np.int64), 0, mx - 1)
    j = np.clip(np.floor(sy).astype(np.int64), 0, my - 1)
    a = sx - i
    b = sy - j
    ll = full[j, i]
    lr = full[j, i + 1]
    ur = full[j + 1, i + 1]
    ul = full[j + 1, i]
    lower = ll + a * (lr - ll) + b * (ur - lr)
    upper = ll + b * (ul - ll) + a * (ur - ul)
    return np.where(a >= b, lower, upper)


def _one(t):
    return 1.0


def _linear(t):
    return t


def _decay(t):
    return math.exp(-t) if np.isscalar(t) else np.exp(-t)


TIME_FACTORS = {"one": _one, "t": _linear, "exp_neg_t": _decay, "zero": None}


@dataclass(frozen=True)
class SeparableP1Source:
    """f(x, y, t) = s(t) * P1-interpolant(g)(x, y); ``kind`` names s."""

    grid: SpatialGrid
    nodal: np.ndarray = field(repr=False)
    kind: str = "one"

    def __post_init__(self):
        if self.kind not in TIME_FACTORS:
            raise ValueError(f"unknown time factor {self.kind!r}")
        g = np.asarray(self.nodal, dtype=float)
        if g.shape != (self.grid.ndof,):
            raise ValueError(f"nodal source must have shape ({self.grid.ndof},)")
        object.__setattr__(self, "nodal", g)

    def time_factor(self, t: float) -> float:
        f = TIME_FACTORS[self.kind]
        return 0.0 if f is None else float(f(t))

    def __call__(self, x, y, t):
        if self.kind == "zero":
            return np.zeros_like(np.asarray(x, dtype=float))
        return self.time_factor(t) * p1_interpolate(self.grid, self.nodal, x, y)


@dataclass(frozen=True)
class NodalInitial:
    """Initial value given by its interior nodal values (stepper.py:149-152)."""

    grid: SpatialGrid
    nodal: np.ndarray = field(repr=False)

    def __call__(self, x, y):
        x = np.asarray(x, dtype=float)
        if x.shape == (self.grid.ndof,):
            gx, gy = self.grid.interior_nodes()
            if np.array_equal(x, gx) and np.array_equal(np.asarray(y, dtype=float), gy):
                return self.nodal.copy()
        return p1_interpolate(self.grid, self.nodal, x, y)
