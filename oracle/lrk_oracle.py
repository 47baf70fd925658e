"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference hot path of arxiv/paper_1703_05638
(package ``lrpostcov``, /root/reference/pkg/src/lrpostcov): the low-rank
factor algebra, the implicit-Euler sweep with SuperLU step solves, the
observation weight, the misfit Hessian apply (IC and source modes), the
factored GMRES, the Arnoldi driver and the SMW posterior variance.  Every
function cites the reference lines it restates.

Pinning: tests/golden/make_golden.py runs the *reference itself* (imported
from /root/reference in the build container) on seeded inputs and stores the
results in tests/golden/*.npz; tests/test_oracle_golden.py checks this module
against those fixtures and against the reference's closed-form known answers
(eigenvector decay, full-observation Hessian eigenvalues).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module, and only as the checker / the timed CPU reference.  The
product package (paper_1703_05638_b200) never imports it.

Third-party arithmetic: numpy (LAPACK geqrf/gesdd/geev/syevd via OpenBLAS)
and scipy.sparse.linalg.splu (SuperLU) — the same libraries the reference
calls (pyproject.toml:10-13 pins numpy>=1.24, scipy>=1.10).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

FLOOR = 1e-15  # lowrank.py:20-22


# ---------------------------------------------------------------- operators
def rotating_upwind(n_side: int, dim: int, w0=(0.0, 0.0, 0.0)):
    """Config C3/C5 convection (extension; unpinned by the reference's tests):
    w(x) = w0 + (2 x2 (1 - x1²), -2 x1 (1 - x2²), 0) upwinded node by node with
    the rule of discretize.py:96-104 (sign of the local wind picks the
    one-sided difference).  Returns the n_x × n_x sparse W (x1 fastest)."""
    n = int(n_side)
    h = 1.0 / (n + 1)
    N = n ** dim
    g = h * (np.arange(n) + 1)
    i = np.arange(N)
    ii = [i % n, (i // n) % n, i // (n * n)]
    x1, x2 = g[ii[0]], g[ii[1]]
    w = [w0[0] + 2 * x2 * (1 - x1**2), w0[1] - 2 * x1 * (1 - x2**2)]
    if dim == 3:
        w.append(np.full(N, float(w0[2])))
    W = sp.lil_matrix((N, N))
    strides = [1, n, n * n]
    for a in range(dim):
        for q in range(N):
            wa = w[a][q]
            if wa > 0:
                W[q, q] += wa / h
                if ii[a][q] > 0:
                    W[q, q - strides[a]] -= wa / h
            elif wa < 0:
                W[q, q] -= wa / h
                if ii[a][q] < n - 1:
                    W[q, q + strides[a]] += wa / h
    return sp.csr_matrix(W)


def fd_operator(n_side: int, kind: str = "heat", nu: float = 1.0, wind=(0.0, 0.0)):
    """5-point FD -Δ, or nu·(5-point) + first-order upwind (discretize.py:90-127).

    Returns (L, h, m_scale) with dofs numbered x1 fastest (discretize.py:3-6).
    """
    n = int(n_side)
    h = 1.0 / (n + 1)
    one = np.ones(n)
    lap1 = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h**2
    eye = sp.identity(n)
    coef = 1.0 if kind == "heat" else nu
    L = coef * (sp.kron(eye, lap1) + sp.kron(lap1, eye))
    if kind != "heat":
        for axis, w in enumerate(wind[:2]):
            if w == 0.0:
                continue
            if w > 0:  # w (u_i - u_{i-1}) / h
                up = (w / h) * sp.diags([-one[1:], one], [-1, 0])
            else:      # -w (u_i - u_{i+1}) / h
                up = (-w / h) * sp.diags([one, -one[1:]], [0, 1])
            L = L + (sp.kron(eye, up) if axis == 0 else sp.kron(up, eye))
    return sp.csr_matrix(L), h, h * h


def galerkin_q1_convection(n_side: int, w0=(0.0, 0.0), rotating: bool = False):
    """Config C3 convection as specified (extension; unpinned by the reference,
    which has first-order upwind only): Galerkin Q1,
    N_ij = ∫ (w·∇φ_j) φ_i, wind at the element centres, assembled element by
    element with explicit 2-point Gauss quadrature of the bilinear shape
    functions (an independent route to the closed-form element matrix the
    device generates on the fly).  Returns N / h² (lumped mass), x1 fastest."""
    n = int(n_side)
    h = 1.0 / (n + 1)
    gp = 0.5 + np.array([-0.5, 0.5]) / np.sqrt(3.0)      # Gauss points on [0, 1]

    def shape(a, t):                                   # 1-D hat on the unit element
        return (1.0 - t, t)[a]

    def dshape(a):
        return (-1.0 / h, 1.0 / h)[a]

    N = sp.lil_matrix((n * n, n * n))
    for p2 in range(-1, n):
        for p1 in range(-1, n):
            xc, yc = h * (p1 + 1.5), h * (p2 + 1.5)
            wx = w0[0] + (2 * yc * (1 - xc**2) if rotating else 0.0)
            wy = w0[1] - (2 * xc * (1 - yc**2) if rotating else 0.0)
            for a2 in (0, 1):
                for a1 in (0, 1):
                    i1, i2 = p1 + a1, p2 + a2
                    if not (0 <= i1 < n and 0 <= i2 < n):
                        continue
                    for b2 in (0, 1):
                        for b1 in (0, 1):
                            j1, j2 = p1 + b1, p2 + b2
                            if not (0 <= j1 < n and 0 <= j2 < n):
                                continue
                            acc = 0.0
                            for s in gp:
                                for t in gp:
                                    phi_i = shape(a1, s) * shape(a2, t)
                                    gx = dshape(b1) * shape(b2, t)
                                    gy = shape(b1, s) * dshape(b2)
                                    acc += 0.25 * h * h * phi_i * (wx * gx + wy * gy)
                            N[i2 * n + i1, j2 * n + j1] += acc
    return sp.csr_matrix(N) / h**2


def config_operator(n_side: int, dim: int = 2, stencil: str = "fd", kind: str = "heat",
                    nu: float = 1.0, wind=(0.0, 0.0, 0.0), wind_field: str = "const"):
    """Config-extension operators (SURVEY §8(c) "Config features beyond the
    reference", Appendix D2; unpinned by the reference's own tests, pinned here
    by closed-form eigenpairs and by golden runs of the unmodified reference
    with these matrices duck-typed in, tests/golden/make_golden.py):
      stencil "q1": L = (K1⊗M1 + M1⊗K1)/h², K1 = (1/h)tridiag(-1,2,-1),
                    M1 = (h/6)tridiag(1,4,1) (Q1 stiffness, lumped mass h²);
      dim 3 "fd":   7-point nu·(-Δ) + first-order upwind per axis.
    Returns (L, h, m_scale) with x1 fastest."""
    if kind != "heat" and stencil == "q1":
        Kq, h, m = config_operator(n_side, 2, "q1", "heat")
        conv = galerkin_q1_convection(n_side, tuple(wind)[:2], wind_field == "rotating")
        return sp.csr_matrix(nu * Kq + conv), h, m
    if kind != "heat" and wind_field == "rotating":
        Ld, h, m = config_operator(n_side, dim, "fd", "heat")
        w3 = tuple(float(v) for v in (tuple(wind) + (0.0,) * 3)[:3])
        return sp.csr_matrix(nu * Ld + rotating_upwind(n_side, dim, w3)), h, m
    if dim == 2 and stencil == "fd":
        return fd_operator(n_side, kind, nu, tuple(wind)[:2])
    n = int(n_side)
    h = 1.0 / (n + 1)
    one = np.ones(n)
    eye = sp.identity(n)
    if stencil == "q1":
        K1 = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h
        M1 = sp.diags([one[1:], 4 * one, one[1:]], [-1, 0, 1]) * (h / 6)
        return sp.csr_matrix((sp.kron(M1, K1) + sp.kron(K1, M1)) / h**2), h, h * h
    coef = 1.0 if kind == "heat" else nu
    axes = []
    for ax in range(3):
        A = coef * sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h**2
        w = float(wind[ax]) if (kind != "heat" and ax < len(wind)) else 0.0
        if w > 0:
            A = A + (w / h) * sp.diags([-one[1:], one], [-1, 0])
        elif w < 0:
            A = A + (-w / h) * sp.diags([one, -one[1:]], [0, 1])
        axes.append(A)
    L = (sp.kron(eye, sp.kron(eye, axes[0])) + sp.kron(eye, sp.kron(axes[1], eye))
         + sp.kron(axes[2], sp.kron(eye, eye)))
    return sp.csr_matrix(L), h, h ** 3


class StepSolver:
    """S = M(I + tau L) factorised once by SuperLU, reused for N and T solves (forward.py:40-68)."""

    def __init__(self, L, m_scale: float, tau: float, n_t: int):
        n_x = L.shape[0]
        self.L = L
        self.m = m_scale
        self.tau = tau
        self.n_x, self.n_t = n_x, n_t
        self.S = (m_scale * (sp.identity(n_x) + tau * L)).tocsc()
        self.lu = spla.splu(self.S)

    def solve(self, B, adjoint=False):
        B = np.asarray(B, dtype=float)
        if B.ndim == 1:
            return self.lu.solve(B[:, None], trans="T" if adjoint else "N")[:, 0]
        return self.lu.solve(B, trans="T" if adjoint else "N")


class CGStepSolver:
    """CPU SUBSTITUTE for StepSolver where SuperLU cannot be set up: the 3-D
    C4/C5 step matrices exhaust memory in splu (MemoryError at 128³
    after > 41 min).  S = M(I + tau L) is SPD for the heat operator, so each
    solve is a CG solve to relative residual 1e-12 (SURVEY §8(d) "extrapolated,
    substitute solver").  Same interface as StepSolver (forward.py:61-68)."""

    def __init__(self, L, m_scale: float, tau: float, n_t: int, rtol: float = 1e-12):
        n_x = L.shape[0]
        self.L = L
        self.m = m_scale
        self.tau = tau
        self.n_x, self.n_t = n_x, n_t
        self.S = sp.csr_matrix(m_scale * (sp.identity(n_x) + tau * L))
        self.rtol = rtol
        self.iterations = 0

    def _one(self, b):
        it = [0]

        def cb(_):
            it[0] += 1
        x, info = spla.cg(self.S, b, rtol=self.rtol, atol=0.0, maxiter=10000, callback=cb)
        if info != 0:
            raise RuntimeError(f"CG step solve did not converge (info {info})")
        self.iterations += it[0]
        return x

    def solve(self, B, adjoint=False):  # S symmetric: S^{-T} = S^{-1}
        B = np.asarray(B, dtype=float)
        if B.ndim == 1:
            return self._one(B)
        return np.column_stack([self._one(B[:, j]) for j in range(B.shape[1])])


class SweepStepper:
    """The sweep of forward.py:133-188 (same arithmetic as ``sweep`` below),
    resumable one time step at a time — the CPU baseline times bounded
    prefixes of an apply with it (bench.py)."""

    def __init__(self, solver, rW1, rW2, eps0, r_max=None, adjoint=False, p=4):
        self.solver, self.eps0, self.r_max, self.adjoint, self.p = solver, eps0, r_max, adjoint, p
        self.rW2 = np.asarray(rW2, float)
        self.B = solver.solve(np.asarray(rW1, float), adjoint)
        n_t = solver.n_t
        self.order = list(range(n_t - 1, -1, -1) if adjoint else range(n_t))
        self.pane = (np.zeros((solver.n_x, 0)), np.zeros((n_t, 0)))
        self.cols, self.idx, self.trace = [], [], []
        self.y = np.zeros(solver.n_x)
        self.count = 0

    @property
    def done(self) -> bool:
        return self.count >= len(self.order)

    def step(self):
        s = self.solver
        k = self.order[self.count]
        self.y = s.solve(s.m * self.y, self.adjoint) + self.B @ self.rW2[k]
        self.cols.append(self.y)
        self.idx.append(k)
        self.count += 1
        if self.count % self.p == 0 or self.done:
            E = np.zeros((s.n_t, len(self.idx)))
            E[self.idx, np.arange(len(self.idx))] = 1.0
            self.pane = truncate(*concat(self.pane, (np.column_stack(self.cols), E)),
                                 self.eps0, self.r_max)
            self.trace.append(self.pane[0].shape[1])
            self.cols.clear()
            self.idx.clear()


# ------------------------------------------------------------ factor algebra
def rank_cut(s, eps0: float, r_max=None) -> int:
    """Smallest r with tail ||s[r:]|| <= eps0 ||s||, after the noise floor (lowrank.py:98-111)."""
    s = np.asarray(s, dtype=float)
    if s.size == 0 or not s[0] > 0:
        return 0
    s = np.where(s < FLOOR * s[0], 0.0, s)
    tail = np.sqrt(np.cumsum((s**2)[::-1]))[::-1]
    keep = int(np.searchsorted(-tail, -eps0 * tail[0], side="left"))
    keep = min(keep, int(np.count_nonzero(s)))
    return keep if r_max is None else min(keep, r_max)


def svd_flip(U, V):
    """Largest-|entry| of each U column made positive (lowrank.py:114-121)."""
    if U.shape[1] == 0:
        return U, V
    rows = np.argmax(np.abs(U), axis=0)
    sgn = np.sign(U[rows, np.arange(U.shape[1])])
    sgn[sgn == 0] = 1.0
    return U * sgn, V * sgn


def truncate(W1, W2, eps0: float, r_max=None):
    """QR both factors, SVD of the core, zero test, rank cut, canonical signs (lowrank.py:124-144)."""
    W1 = np.asarray(W1, float)
    W2 = np.asarray(W2, float)
    n_x, n_t = W1.shape[0], W2.shape[0]
    if W1.shape[1] == 0:
        return np.zeros((n_x, 0)), np.zeros((n_t, 0))
    Q1, R1 = np.linalg.qr(W1)
    Q2, R2 = np.linalg.qr(W2)
    U, s, Vt = np.linalg.svd(R1 @ R2.T)
    if s.size == 0 or s[0] <= FLOOR * np.linalg.norm(R1) * np.linalg.norm(R2):
        return np.zeros((n_x, 0)), np.zeros((n_t, 0))
    r = rank_cut(s, eps0, r_max)
    if r == 0:
        return np.zeros((n_x, 0)), np.zeros((n_t, 0))
    U1, V1 = svd_flip(Q1 @ U[:, :r], Q2 @ Vt[:r].T)
    return U1, V1 * s[:r]


def concat(A, B):
    """lr_add (lowrank.py:147-154): exact sum by concatenation."""
    if A[0].shape[1] == 0:
        return B
    if B[0].shape[1] == 0:
        return A
    return np.hstack([A[0], B[0]]), np.hstack([A[1], B[1]])


def scale(A, c):
    """lr_scale (lowrank.py:157-160)."""
    if c == 0.0:
        return np.zeros((A[0].shape[0], 0)), np.zeros((A[1].shape[0], 0))
    return A[0], A[1] * c


def dot(A, B) -> float:
    """lr_dot (lowrank.py:163-168)."""
    if A[0].shape[1] == 0 or B[0].shape[1] == 0:
        return 0.0
    return float(np.sum((A[0].T @ B[0]) * (A[1].T @ B[1])))


def norm(A) -> float:
    return math.sqrt(max(dot(A, A), 0.0))


def singular_values(A):
    if A[0].shape[1] == 0:
        return np.zeros(0)
    return np.linalg.svd(np.linalg.qr(A[0], mode="r") @ np.linalg.qr(A[1], mode="r").T,
                         compute_uv=False)


# ----------------------------------------------------------------- forward
def apply_K(solver: StepSolver, W1, W2, adjoint=False):
    """K (or Kᵀ) on factors, rank 2r (forward.py:70-95)."""
    if W1.shape[1] == 0:
        return W1, W2
    S = solver.S.T if adjoint else solver.S
    shifted = np.zeros_like(W2)
    if adjoint:
        shifted[:-1] = W2[1:]
    else:
        shifted[1:] = W2[:-1]
    return np.hstack([S @ W1, -solver.m * W1]), np.hstack([W2, shifted])


def sweep(solver: StepSolver, rW1, rW2, eps0, r_max=None, adjoint=False, p=4):
    """Time substitution with a flush every p steps (forward.py:133-188).

    Returns (W1, W2, trace) where trace is the pane rank after each flush plus
    the final rank (forward.py:175, :187).
    """
    n_x, n_t = solver.n_x, solver.n_t
    rW1 = np.asarray(rW1, float)
    rW2 = np.asarray(rW2, float)
    if rW1.shape[1] == 0:
        return np.zeros((n_x, 0)), np.zeros((n_t, 0)), []
    B = solver.solve(rW1, adjoint)
    order = range(n_t - 1, -1, -1) if adjoint else range(n_t)
    pane = (np.zeros((n_x, 0)), np.zeros((n_t, 0)))
    cols, idx, trace = [], [], []
    y = np.zeros(n_x)

    def fold(pane):
        E = np.zeros((n_t, len(idx)))
        E[idx, np.arange(len(idx))] = 1.0
        out = truncate(*concat(pane, (np.column_stack(cols), E)), eps0, r_max)
        trace.append(out[0].shape[1])
        cols.clear()
        idx.clear()
        return out

    for count, k in enumerate(order, 1):
        y = solver.solve(solver.m * y, adjoint) + B @ rW2[k]
        cols.append(y)
        idx.append(k)
        if count % p == 0:
            pane = fold(pane)
    if cols:
        pane = fold(pane)
    trace.append(pane[0].shape[1])
    return pane[0], pane[1], trace


def gmres(solver: StepSolver, rW1, rW2, eps0, r_max=None, adjoint=False, tol=1e-8,
          max_iter=None):
    """Block-preconditioned GMRES on factored iterates (forward.py:204-274).

    Returns ((W1, W2), iterations, trace); raises RuntimeError on stagnation.
    """
    def pre(A):
        return (solver.solve(A[0], adjoint), A[1]) if A[0].shape[1] else A

    if max_iter is None:
        max_iter = solver.n_t + 5
    b = truncate(*pre((rW1, rW2)), eps0, r_max)
    beta = norm(b)
    if beta == 0.0:
        return (np.zeros((solver.n_x, 0)), np.zeros((solver.n_t, 0))), 0, []
    V = [scale(b, 1.0 / beta)]
    H = np.zeros((max_iter + 1, max_iter))
    trace = []
    for j in range(max_iter):
        w = truncate(*pre(apply_K(solver, *V[j], adjoint)), eps0, r_max)
        for i in range(j + 1):
            H[i, j] = dot(w, V[i])
            w = concat(w, scale(V[i], -H[i, j]))
        w = truncate(*w, eps0, r_max)
        H[j + 1, j] = norm(w)
        trace.append(w[0].shape[1])
        e1 = np.zeros(j + 2)
        e1[0] = beta
        y = np.linalg.lstsq(H[: j + 2, : j + 1], e1, rcond=None)[0]
        resid = float(np.linalg.norm(H[: j + 2, : j + 1] @ y - e1)) / beta
        if resid <= tol or H[j + 1, j] <= 1e-14 * max(1.0, float(np.abs(H[: j + 2, : j + 1]).max())):
            x = (np.zeros((solver.n_x, 0)), np.zeros((solver.n_t, 0)))
            for i in range(j + 1):
                x = concat(x, scale(V[i], float(y[i])))
            return truncate(*x, eps0, r_max), j + 1, trace
        V.append(scale(w, 1.0 / H[j + 1, j]))
    raise RuntimeError(f"GMRES stagnated after {max_iter} iterations (residual {resid:.3e})")


# ----------------------------------------------------------------- Hessian
class Problem:
    """Bundle of everything one Hessian apply needs (HessianContext, hessian.py:159-187)."""

    def __init__(self, n_side, n_t, mask, beta_noise, gamma_prior, eps0=1e-8, r_max=None,
                 kind="heat", nu=1.0, wind=(0.0, 0.0), T=1.0, compress_every=4, dim=2,
                 stencil="fd", prior=None, obs_every=1, wind_field="const"):
        L, h, m = config_operator(n_side, dim, stencil, kind, nu, wind, wind_field)
        self.n_side, self.h, self.m = n_side, h, m
        self.tau = T / n_t
        self.solver = StepSolver(L, m, self.tau, n_t)
        self.mask = np.asarray(mask, bool)
        self.beta_noise = beta_noise
        self.gamma = gamma_prior
        self.eps0, self.r_max, self.p = eps0, r_max, compress_every
        self.weight = beta_noise * self.tau * m  # hessian.py:153
        self.obs_every = int(obs_every)
        # config prior sqrt: sqrt(gamma) (delta I + gamma_p L)^{-1}
        self.prior_lu = None
        if prior is not None:
            delta, gp = prior
            # L_Δ: the PDE's own discrete Laplacian (its diffusion part, without ν or wind)
            Ld = L if kind == "heat" else config_operator(n_side, dim, stencil, "heat")[0]
            self.prior_lu = spla.splu((delta * sp.identity(L.shape[0]) + gp * Ld).tocsc())

    def prior_sqrt(self, x):
        """Γ^{1/2} x: sqrt(γ)·x (hessian.py:215) or sqrt(γ)(δI+γ_pL)⁻¹x (config prior)."""
        x = math.sqrt(self.gamma) * np.asarray(x, float)
        if self.prior_lu is None:
            return x
        return self.prior_lu.solve(x if x.ndim == 2 else x[:, None]).reshape(x.shape)

    def observe(self, W1, W2):
        """Mask + weight + truncate (hessian.py:138-156); time-row mask of
        time-subsampled sensors before the truncation."""
        if W1.shape[1] == 0:
            return W1, W2
        Z1 = np.where(self.mask[:, None], W1, 0.0) * self.weight
        if self.obs_every > 1:
            keep = (np.arange(W2.shape[0]) + 1) % self.obs_every == 0
            W2 = np.where(keep[:, None], W2, 0.0)
        return truncate(Z1, W2, self.eps0, self.r_max)


def hessian_ic(P: Problem, v):
    """H̃ v for the IC parameter (hessian.py:211-226); returns (out, max_rank)."""
    n_t = P.solver.n_t
    e0 = np.zeros((n_t, 1))
    e0[0, 0] = 1.0
    Y1, Y2, tr1 = sweep(P.solver, (P.m * P.prior_sqrt(v))[:, None], e0, P.eps0, P.r_max,
                        False, P.p)
    Z1, Z2 = P.observe(Y1, Y2)
    Q1, Q2, tr2 = sweep(P.solver, Z1, Z2, P.eps0, P.r_max, True, P.p)
    out = P.m * (Q1 @ Q2[0]) if Q1.shape[1] else np.zeros(P.solver.n_x)
    return P.prior_sqrt(out), max(tr1 + [Z1.shape[1]] + tr2)


def hessian_st(P: Problem, V1, V2):
    """H̃ vec(v) for the space-time source (hessian.py:229-245); returns ((W1, W2), max_rank)."""
    inj = P.tau * P.m  # forward.py:118-122
    r1 = P.prior_sqrt(np.asarray(V1, float))
    r1, r2 = scale((r1, np.asarray(V2, float)), inj)
    Y1, Y2, tr1 = sweep(P.solver, r1, r2, P.eps0, P.r_max, False, P.p)
    Z1, Z2 = P.observe(Y1, Y2)
    Q1, Q2, tr2 = sweep(P.solver, Z1, Z2, P.eps0, P.r_max, True, P.p)
    out = truncate(*scale((P.prior_sqrt(Q1) if Q1.shape[1] else Q1, Q2), inj), P.eps0, P.r_max)
    return out, max(tr1 + [Z1.shape[1]] + tr2 + [out[0].shape[1]])


# ------------------------------------------------------------------ Arnoldi
def arnoldi_dense(apply, v1, m_a, eps_eig=1e-1, check_every=10, rtol=1e-3):
    """Dense-vector Arnoldi with MGS2 (arnoldi.py:271-375, on_breakdown='stop').

    Returns (H, basis, ritz_values, iterations).
    """
    v1 = np.asarray(v1, float)
    basis = [v1 / np.linalg.norm(v1)]
    H = np.zeros((m_a + 1, m_a))
    prev = None
    done = 0
    for j in range(m_a):
        w = np.asarray(apply(basis[j]), float)
        for _ in range(2):
            for i in range(j + 1):
                hij = float(w @ basis[i])
                H[i, j] += hij
                w = w - hij * basis[i]
        h = float(np.linalg.norm(w))
        H[j + 1, j] = h
        done = j + 1
        if h <= 1e-14:
            break
        basis.append(w / h)
        if (j + 1) % check_every == 0 and j + 1 < m_a:
            vals = np.linalg.eigvals(H[: j + 1, : j + 1])
            vals = vals[np.argsort(-vals.real)]
            if prev is not None and _stable(vals, prev, eps_eig, rtol):
                break
            prev = vals
    Hm = H[:done, :done]
    vals = np.linalg.eigvals(Hm)
    return H[: done + 1, :done], basis, vals[np.argsort(-vals.real)], done


def _stable(vals, prev, eps_eig, rtol):
    """_stop_ready (arnoldi.py:242-268)."""
    above = int(np.sum(vals.real >= eps_eig))
    if above != int(np.sum(prev.real >= eps_eig)):
        return False
    n_check = above if above > 0 else min(1, len(vals), len(prev))
    if n_check > len(prev):
        return False
    for i in range(n_check):
        d = max(abs(vals[i].real), abs(prev[i].real), 1e-300)
        if abs(vals[i].real - prev[i].real) / d > rtol:
            return False
    return True


def ritz_vectors(H, basis):
    """Ritz combination with the symmetric path of arnoldi.py:197-212."""
    m = H.shape[1]
    Hm = H[:m, :m]
    vals, vecs = np.linalg.eig(Hm)
    order = np.argsort(-vals.real)
    vals, vecs = vals[order], vecs[:, order]
    sc = float(np.abs(Hm).max()) if m else 0.0
    if sc > 0 and float(np.abs(Hm - Hm.T).max()) <= 1e-6 * sc:
        vecs = np.linalg.eigh(0.5 * (Hm + Hm.T))[1][:, ::-1]
    B = np.column_stack(basis[:m])
    out = []
    for i in range(m):
        x = B @ np.real(vecs[:, i])
        out.append(x / np.linalg.norm(x))
    return vals, out


def posterior_variance(vals, vecs, gamma, eps_eig, prior_matrix=None):
    """SMW variance diag γ(1 - Σ λ̃ v²) with QR re-orthonormalisation (posterior.py:56-111).
    Config prior: prior_matrix = dense P = (δI+γ_pL)⁻¹ and
    diag = γ(diag(P²) - Σ λ̃ (P v)²)."""
    real = np.asarray(vals).real
    keep = [i for i in np.argsort(-real) if real[i] >= eps_eig]
    base = 1.0 if prior_matrix is None else np.sum(prior_matrix * prior_matrix, axis=0)
    if not keep:
        return gamma * base * np.ones(len(vecs[0]))
    V = np.column_stack([vecs[i] / np.linalg.norm(vecs[i]) for i in keep])
    V = np.linalg.qr(V)[0]
    if prior_matrix is not None:
        V = prior_matrix @ V
    lam = real[keep]
    return gamma * (base - (V**2) @ (lam / (lam + 1.0)))


# ------------------------------------------------------------- closed forms
def fd_eig(m, n, n_side):
    """(4/h²)(sin²(mπh/2) + sin²(nπh/2)) (discretize.py:137-144)."""
    h = 1.0 / (n_side + 1)
    return 4.0 / h**2 * (math.sin(m * math.pi * h / 2) ** 2 + math.sin(n * math.pi * h / 2) ** 2)


def fd_eigvec(m, n, n_side):
    """Unit dense FD eigenvector, x1 fastest (discretize.py:147-168)."""
    x = np.arange(1, n_side + 1) / (n_side + 1)
    f1 = np.sin(m * math.pi * x)
    f2 = np.sin(n * math.pi * x)
    return np.kron(f2 / np.linalg.norm(f2), f1 / np.linalg.norm(f1))


def ic_eigenvalue_full_obs(m, n, n_side, n_t, beta_noise, gamma, T=1.0):
    """μ = γ β τ M Σ_{k=1}^{n_t} θ^{2k} on FD eigenvectors (test_hessian.py:129-139)."""
    h = 1.0 / (n_side + 1)
    tau = T / n_t
    theta = 1.0 / (1.0 + tau * fd_eig(m, n, n_side))
    return gamma * beta_noise * tau * h * h * sum(theta ** (2 * k) for k in range(1, n_t + 1))


def config_eig(modes, n_side, stencil="fd"):
    """Eigenvalue of the config L on a separable DST-I mode."""
    h = 1.0 / (n_side + 1)
    ms = np.asarray(modes, float)
    if stencil == "q1":
        c = np.cos(ms * math.pi * h)
        k1, m1 = (2 / h) * (1 - c), (h / 3) * (2 + c)
        return float((k1[0] * m1[1] + m1[0] * k1[1]) / h**2)
    s_ = np.sin(ms * math.pi * h / 2)
    return float(4.0 / h**2 * np.sum(s_ * s_))


def config_eigvec(modes, n_side):
    """Unit separable DST-I eigenvector (x1 fastest) in 2-D or 3-D."""
    x = np.arange(1, n_side + 1) / (n_side + 1)
    v = np.ones(1)
    for m in modes:  # x1 first -> innermost
        f = np.sin(m * math.pi * x)
        v = np.kron(f / np.linalg.norm(f), v)
    return v


def config_ic_eigenvalue(modes, n_side, n_t, beta_noise, gamma=1.0, stencil="fd", prior=None,
                         obs_every=1, T=1.0):
    """Full-observation IC Hessian eigenvalue on a DST-I mode, generalising
    test_hessian.py:129-139: μ = γ β τ M Σ_{k observed} θ^{2k} · (δ+γ_p λ)⁻²."""
    d = len(modes)
    h = 1.0 / (n_side + 1)
    tau = T / n_t
    lam = config_eig(modes, n_side, stencil)
    theta = 1.0 / (1.0 + tau * lam)
    ks = [k for k in range(1, n_t + 1) if k % obs_every == 0]
    mu = gamma * beta_noise * tau * h**d * sum(theta ** (2 * k) for k in ks)
    if prior is not None:
        mu /= (prior[0] + prior[1] * lam) ** 2
    return mu
