"""Grids and discrete operators (host-side setup; mirrors lrpostcov/discretize.py).

Unit square, homogeneous Dirichlet data, interior dofs numbered with x1
fastest (discretize.py:3-6), lumped mass M = h^d (discretize.py:33-34).
The device path never reads the assembled matrix: the sweep uses the DST-I
eigen-decomposition of the heat stencil and the SpMM kernel generates the
5-point coefficients on the fly.  `L` is still assembled (scipy CSR) for
API compatibility (SpatialOperator.L, discretize.py:46-62).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import InvalidConfigError


@dataclass(frozen=True)
class Grid:
    """Uniform interior lattice of the unit square (discretize.py:19-43)."""

    n_side: int
    h: float
    d: int = 2

    @property
    def n_x(self) -> int:
        return self.n_side ** self.d

    @property
    def m_scale(self) -> float:
        return self.h ** self.d

    def ij_to_dof(self, i: int, j: int) -> int:
        return j * self.n_side + i

    def dof_to_ij(self, k: int) -> tuple[int, int]:
        return k % self.n_side, k // self.n_side

    def coords(self):
        axis = self.h * (1 + np.arange(self.n_side))
        return np.tile(axis, self.n_side), np.repeat(axis, self.n_side)


@dataclass(frozen=True)
class TimeGrid:
    n_t: int
    tau: float
    T: float = 1.0


@dataclass(frozen=True)
class SpatialOperator:
    """-Δ (heat) or -nu Δ + wind·∇ (convdiff) with zero Dirichlet data."""

    kind: str
    grid: Grid
    L: sp.csr_matrix
    nu: float = 1.0
    wind: tuple[float, float] = (0.0, 0.0)

    @property
    def m_scale(self) -> float:
        return self.grid.m_scale


def build_grid(n_side: int) -> Grid:
    if n_side < 2:
        raise InvalidConfigError(f"n_side must be >= 2, got {n_side}")
    return Grid(n_side=int(n_side), h=1.0 / (n_side + 1))


def build_time_grid(n_t: int, T: float = 1.0) -> TimeGrid:
    if n_t < 1 or T <= 0:
        raise InvalidConfigError(f"need n_t >= 1 and T > 0, got n_t={n_t}, T={T}")
    return TimeGrid(n_t=int(n_t), tau=T / n_t, T=T)


def stencil_coefficients(kind: str, h: float, nu: float = 1.0, wind=(0.0, 0.0)):
    """(centre, west, east, south, north) of the 5-point operator row.

    Heat: 4/h² centre, -1/h² neighbours (discretize.py:90-112).  Convdiff adds
    first-order upwind along each axis by the sign of the wind component
    (discretize.py:96-104, :115-127).
    """
    ih2 = 1.0 / (h * h)
    scale = 1.0 if kind == "heat" else float(nu)
    cc, cw, ce, cs, cn = 4 * scale * ih2, -scale * ih2, -scale * ih2, -scale * ih2, -scale * ih2
    if kind != "heat":
        w1, w2 = float(wind[0]), float(wind[1])
        if w1 > 0:
            cc, cw = cc + w1 / h, cw - w1 / h
        elif w1 < 0:
            cc, ce = cc - w1 / h, ce + w1 / h
        if w2 > 0:
            cc, cs = cc + w2 / h, cs - w2 / h
        elif w2 < 0:
            cc, cn = cc - w2 / h, cn + w2 / h
    return cc, cw, ce, cs, cn


def _assemble(grid: Grid, coeffs) -> sp.csr_matrix:
    n = grid.n_side
    cc, cw, ce, cs, cn = coeffs
    i1 = np.tile(np.arange(n), n)
    diags = [np.full(n * n, cc)]
    offsets = [0]
    west = np.where(i1[1:] > 0, cw, 0.0)       # entry (k, k-1) valid when i1(k) > 0
    east = np.where(i1[:-1] < n - 1, ce, 0.0)  # entry (k, k+1) valid when i1(k) < n-1
    diags += [west, east, np.full(n * n - n, cs), np.full(n * n - n, cn)]
    offsets += [-1, 1, -n, n]
    return sp.diags(diags, offsets, shape=(n * n, n * n), format="csr")


def assemble_heat(grid: Grid) -> SpatialOperator:
    return SpatialOperator(kind="heat", grid=grid, L=_assemble(grid, stencil_coefficients("heat", grid.h)))


def assemble_convdiff(grid: Grid, nu: float, wind) -> SpatialOperator:
    if nu <= 0:
        raise InvalidConfigError(f"viscosity nu must be positive, got {nu}")
    w = (float(wind[0]), float(wind[1]))
    L = _assemble(grid, stencil_coefficients("convdiff", grid.h, nu, w))
    return SpatialOperator(kind="convdiff", grid=grid, L=L, nu=float(nu), wind=w)


def analytic_poisson_eig(m: int, n: int, a: float = 1.0, b: float = 1.0) -> float:
    if m < 1 or n < 1 or a <= 0 or b <= 0:
        raise InvalidConfigError("need m,n >= 1 and a,b > 0")
    return float(np.pi ** 2 * ((m / a) ** 2 + (n / b) ** 2))


def _check_mode(m, n, grid):
    if not (1 <= m <= grid.n_side and 1 <= n <= grid.n_side):
        raise InvalidConfigError(f"mode indices must lie in [1, {grid.n_side}], got ({m}, {n})")


def discrete_fd_eig(m: int, n: int, grid: Grid) -> float:
    """(4/h²)(sin²(mπh/2) + sin²(nπh/2)) — discretize.py:137-144."""
    _check_mode(m, n, grid)
    s = np.sin(np.array([m, n]) * np.pi * grid.h / 2)
    return float(4.0 / grid.h ** 2 * np.sum(s * s))


def analytic_separable_eigvec(m: int, n: int, grid: Grid):
    _check_mode(m, n, grid)
    x = grid.h * (1 + np.arange(grid.n_side))
    f1, f2 = np.sin(m * np.pi * x), np.sin(n * np.pi * x)
    return f1 / np.linalg.norm(f1), f2 / np.linalg.norm(f2)


def eigvec_dense(m: int, n: int, grid: Grid) -> np.ndarray:
    f1, f2 = analytic_separable_eigvec(m, n, grid)
    return np.kron(f2, f1)
