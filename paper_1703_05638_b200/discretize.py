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
        if self.d == 3:
            n = self.n_side
            return (np.tile(axis, n * n), np.tile(np.repeat(axis, n), n), np.repeat(axis, n * n))
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
    wind: tuple = (0.0, 0.0)
    stencil: str = "fd"   # "fd" (reference 5-point / 3-D 7-point) or "q1" (Q1-lumped 9-point)
    wind_field: str = "const"  # "const" (reference) or "rotating" (configs C3/C5)

    @property
    def m_scale(self) -> float:
        return self.grid.m_scale


def build_grid(n_side: int, d: int = 2) -> Grid:
    if n_side < 2:
        raise InvalidConfigError(f"n_side must be >= 2, got {n_side}")
    if d not in (2, 3):
        raise InvalidConfigError(f"dimension must be 2 or 3, got {d}")
    return Grid(n_side=int(n_side), h=1.0 / (n_side + 1), d=int(d))


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


def _lap1(n: int, h: float):
    one = np.ones(n)
    return sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h**2


def _upwind1(n: int, h: float, w: float):
    """First-order upwind w·d/dx by the sign of w (discretize.py:96-104)."""
    one = np.ones(n)
    if w > 0:
        return (w / h) * sp.diags([-one[1:], one], [-1, 0])
    if w < 0:
        return (-w / h) * sp.diags([one, -one[1:]], [0, 1])
    return sp.csr_matrix((n, n))


def _assemble_3d(grid: Grid, nu: float = 1.0, wind=(0.0, 0.0, 0.0)) -> sp.csr_matrix:
    """3-D 7-point FD nu·(-Δ) + per-axis upwind, x1 fastest (config C4/C5 extension)."""
    n, h = grid.n_side, grid.h
    eye = sp.identity(n)
    ops = [nu * _lap1(n, h) + _upwind1(n, h, float(w)) for w in (tuple(wind) + (0.0,) * 3)[:3]]
    return sp.csr_matrix(sp.kron(eye, sp.kron(eye, ops[0])) + sp.kron(eye, sp.kron(ops[1], eye))
                         + sp.kron(ops[2], sp.kron(eye, eye)))


def _assemble_q1(grid: Grid) -> sp.csr_matrix:
    """Q1 bilinear stiffness with lumped mass, L = K_Q1 / h²:
    K_Q1 = K1 ⊗ M1 + M1 ⊗ K1, K1 = (1/h)[-1 2 -1], M1 = (h/6)[1 4 1]; the
    9-point stencil has centre 8/3 and all eight neighbours -1/3 (times 1/h²)."""
    n, h = grid.n_side, grid.h
    one = np.ones(n)
    K1 = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h
    M1 = sp.diags([one[1:], 4 * one, one[1:]], [-1, 0, 1]) * (h / 6)
    return sp.csr_matrix((sp.kron(K1, M1) + sp.kron(M1, K1)) / h**2)


def assemble_heat(grid: Grid, stencil: str = "fd") -> SpatialOperator:
    if stencil not in ("fd", "q1"):
        raise InvalidConfigError(f"unknown stencil {stencil!r}")
    if stencil == "q1":
        if grid.d != 2:
            raise InvalidConfigError("the Q1-lumped stencil is 2-D")
        return SpatialOperator(kind="heat", grid=grid, L=_assemble_q1(grid), stencil="q1")
    if grid.d == 3:
        return SpatialOperator(kind="heat", grid=grid, L=_assemble_3d(grid))
    return SpatialOperator(kind="heat", grid=grid, L=_assemble(grid, stencil_coefficients("heat", grid.h)))


def rotating_wind(grid: Grid, w0=(0.0, 0.0, 0.0)):
    """Per-node wind of configs C3/C5: w0 + (2 x2 (1 - x1²), -2 x1 (1 - x2²), 0)."""
    c = grid.coords()
    x1, x2 = c[0], c[1]
    w0 = tuple(float(v) for v in (tuple(w0) + (0.0,) * 3)[:3])
    W = [w0[0] + 2 * x2 * (1 - x1**2), w0[1] - 2 * x1 * (1 - x2**2)]
    if grid.d == 3:
        W.append(np.full(grid.n_x, w0[2]))
    return W


def _upwind_field(grid: Grid, W) -> sp.csr_matrix:
    """First-order upwind by the sign of the LOCAL wind (discretize.py:96-104
    applied node by node): row q gets |w_a(q)|/h on the diagonal and
    -|w_a(q)|/h on its upstream neighbour along each axis."""
    n, N, h = grid.n_side, grid.n_x, grid.h
    idx = np.arange(N)
    comp = [idx % n, (idx // n) % n, idx // (n * n)]
    stride = [1, n, n * n]
    rows, cols, vals = [idx], [idx], [np.sum([np.abs(w) for w in W], axis=0) / h]
    for a, w in enumerate(W):
        m = (w > 0) & (comp[a] > 0)
        rows.append(idx[m]); cols.append(idx[m] - stride[a]); vals.append(-w[m] / h)
        m = (w < 0) & (comp[a] < n - 1)
        rows.append(idx[m]); cols.append(idx[m] + stride[a]); vals.append(w[m] / h)
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(N, N))


def _galerkin_q1_convection(grid: Grid, w0, rotating: bool) -> sp.csr_matrix:
    """Galerkin Q1 convection N_ij = ∫ (w·∇φ_j) φ_i on the uniform grid, the wind
    taken at the element centres (w0, plus the rotating field of config C3),
    divided by the lumped mass h².  Per element with
    lower-left node p and local nodes a, b in {0,1}²:
    N^e_ab = h [ w_x (s_b1/2) m(a2,b2) + w_y m(a1,b1) (s_b2/2) ], s = (-1, +1),
    m(equal) = 1/3, m(different) = 1/6."""
    n, h = grid.n_side, grid.h
    p = np.arange(-1, n)
    p1, p2 = np.meshgrid(p, p, indexing="xy")      # p1 along axis 1 (x1 fastest when flattened)
    xc, yc = h * (p1 + 1.5), h * (p2 + 1.5)
    wx = w0[0] + (2 * yc * (1 - xc**2) if rotating else 0.0) + 0.0 * xc
    wy = w0[1] - (2 * xc * (1 - yc**2) if rotating else 0.0) + 0.0 * xc
    rows, cols, vals = [], [], []
    for a2 in (0, 1):
        for a1 in (0, 1):
            for b2 in (0, 1):
                for b1 in (0, 1):
                    m1 = 1 / 3 if a1 == b1 else 1 / 6
                    m2 = 1 / 3 if a2 == b2 else 1 / 6
                    ne = h * (wx * (0.5 if b1 else -0.5) * m2 + wy * m1 * (0.5 if b2 else -0.5))
                    ia1, ia2, ib1, ib2 = p1 + a1, p2 + a2, p1 + b1, p2 + b2
                    ok = ((ia1 >= 0) & (ia1 < n) & (ia2 >= 0) & (ia2 < n)
                          & (ib1 >= 0) & (ib1 < n) & (ib2 >= 0) & (ib2 < n))
                    rows.append((ia2 * n + ia1)[ok])
                    cols.append((ib2 * n + ib1)[ok])
                    vals.append(ne[ok])
    N = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(grid.n_x, grid.n_x))
    return N / h**2


def assemble_convdiff(grid: Grid, nu: float, wind, field: str = "const",
                      scheme: str = "upwind") -> SpatialOperator:
    """-nu Δ + w·∇ with first-order upwind (discretize.py:115-127).  field
    "rotating" (config extension) adds the C3/C5 rotating field to `wind` and
    upwinds node by node.  scheme "galerkin" (config C3 as specified, SURVEY
    Appendix D3: Q1 FEM whose SUPG parameter vanishes because the element
    Péclet number |w| h / (2 nu) is below one) is the 2-D Q1 stiffness plus the
    Galerkin Q1 convection matrix, lumped mass."""
    if nu <= 0:
        raise InvalidConfigError(f"viscosity nu must be positive, got {nu}")
    if field not in ("const", "rotating"):
        raise InvalidConfigError(f"unknown wind field {field!r}")
    if scheme not in ("upwind", "galerkin"):
        raise InvalidConfigError(f"unknown convection scheme {scheme!r}")
    if scheme == "galerkin":
        if grid.d != 2:
            raise InvalidConfigError("the Galerkin Q1 operator is 2-D")
        w2 = (float(wind[0]), float(wind[1]))
        L = sp.csr_matrix(float(nu) * _assemble_q1(grid)
                          + _galerkin_q1_convection(grid, w2, field == "rotating"))
        return SpatialOperator(kind="convdiff", grid=grid, L=L, nu=float(nu), wind=w2,
                               stencil="q1", wind_field=field)
    if field == "rotating":
        w3 = tuple(float(x) for x in (tuple(wind) + (0.0,) * 3)[:3])
        lap = _assemble_3d(grid, float(nu)) if grid.d == 3 else \
            float(nu) * _assemble(grid, stencil_coefficients("heat", grid.h))
        L = sp.csr_matrix(lap + _upwind_field(grid, rotating_wind(grid, w3)))
        return SpatialOperator(kind="convdiff", grid=grid, L=L, nu=float(nu),
                               wind=w3 if grid.d == 3 else w3[:2], wind_field="rotating")
    if grid.d == 3:
        w3 = tuple(float(x) for x in (tuple(wind) + (0.0,) * 3)[:3])
        return SpatialOperator(kind="convdiff", grid=grid, L=_assemble_3d(grid, float(nu), w3),
                               nu=float(nu), wind=w3)
    w = (float(wind[0]), float(wind[1]))
    L = _assemble(grid, stencil_coefficients("convdiff", grid.h, nu, w))
    return SpatialOperator(kind="convdiff", grid=grid, L=L, nu=float(nu), wind=w)


def operator_eig(grid: Grid, modes, stencil: str = "fd") -> float:
    """Eigenvalue of L on the separable DST-I mode `modes` (1-based, one per
    axis): FD sum of (4/h²)sin²(mπh/2); Q1-lumped [k1(m)m1(n) + m1(m)k1(n)]/h²
    with k1 = (2/h)(1 - cos mπh), m1 = (h/3)(2 + cos mπh)."""
    h = grid.h
    ms = np.asarray(modes, dtype=float)
    if ms.size != grid.d or np.any(ms < 1) or np.any(ms > grid.n_side):
        raise InvalidConfigError(f"need {grid.d} mode indices in [1, {grid.n_side}]")
    if stencil == "q1":
        c = np.cos(ms * np.pi * h)
        k1, m1 = (2 / h) * (1 - c), (h / 3) * (2 + c)
        return float((k1[0] * m1[1] + m1[0] * k1[1]) / h**2)
    s = np.sin(ms * np.pi * h / 2)
    return float(4.0 / h**2 * np.sum(s * s))


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


def eigvec_dense(m: int, n: int, grid: Grid, k: int | None = None) -> np.ndarray:
    f1, f2 = analytic_separable_eigvec(m, n, grid)
    if grid.d == 3:
        if k is None or not (1 <= k <= grid.n_side):
            raise InvalidConfigError("3-D eigenvectors need a third mode index")
        x = grid.h * (1 + np.arange(grid.n_side))
        f3 = np.sin(k * np.pi * x)
        return np.kron(f3 / np.linalg.norm(f3), np.kron(f2, f1))
    return np.kron(f2, f1)


# ------------------------------------------------------------------- text exchange
def export_coo(op: SpatialOperator, path) -> None:
    """One 'row col value' line per stored entry, 0-based, 17 significant digits
    (discretize.py:171-176): the assembled matrix for use outside the package."""
    m = sp.coo_matrix(op.L)
    with open(path, "w") as fh:
        fh.writelines(f"{int(i)} {int(j)} {float(v):.17g}\n" for i, j, v in zip(m.row, m.col, m.data))


def import_coo(path, n: int) -> sp.csr_matrix:
    """Inverse of export_coo (discretize.py:179-190); blank lines are skipped."""
    triples = [line.split() for line in open(path) if line.strip()]
    if not triples:
        return sp.csr_matrix((n, n))
    r, c, v = zip(*triples)
    return sp.csr_matrix((np.array(v, dtype=float), (np.array(r, dtype=int), np.array(c, dtype=int))),
                         shape=(n, n))
