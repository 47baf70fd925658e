"""Config-scale golden fixtures, produced by running the REFERENCE package itself.

Run in the build container (the reference is mounted read-only there; it is
absent on the GPU box, so its outputs travel as .npz files):

    python tests/golden/make_golden_config.py [case ...]   # default: all cases

Cases (BASELINE.json configs):
  c2_apply   — ONE IC Hessian apply at the exact bench configuration C2
               (Q1-lumped 256², n_t 512, 32×32 point sensors, σ 0.01 → w = 1/σ²,
               prior (I + 0.05 L)⁻¹ on each side, eps0 1e-8, r_max 32) with the
               per-flush rank traces of both sweeps (hessian.py:211-226).
  c2_arnoldi — the C2 eigen run: lr_arnoldi with the reference's default stop
               rule (m_a 50, eps_eig 0.1, check_every 10; arnoldi.py:271-375,
               cli.py:58-60), seeded start (cli.py:247-266, seed 1), then
               build_summary (posterior.py:65-111) and the pointwise variance
               with the config prior γ[diag(P²) − Σ λ̃ (P v)²].
  c1_source  — C1: source mode (hessian.py:229-245), Q1-lumped 32², n_t 64, all
               nodes observed, σ 0.01, prior (I + 0.1 L)⁻¹, r_max 20, low-rank
               Arnoldi m_a 10 from the seeded rank-1 start (cli.py:250-262, seed 0).
  c4_sweep3d — the C4 path at n_x ≥ 1e5: 3-D 7-point heat 48³ (n_x 110,592),
               n_t 32, 12³ point sensors every 4th step, σ 0.005, prior
               (I + 0.02 L)⁻¹, r_max 64; one IC apply with rank traces.

The reference pipeline is UNMODIFIED: the config matrices are duck-typed into
SpaceTimeOperator, and the prior / time-row mask wrap misfit_apply_ic /
misfit_apply_st line by line, exactly as make_golden.py's cfg_*
cases.  Each case writes tests/golden/config_<case>.npz.
"""

from __future__ import annotations

import math
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def q1_matrix(n, h):
    import scipy.sparse as sp
    one = np.ones(n)
    K1 = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h
    M1 = sp.diags([one[1:], 4 * one, one[1:]], [-1, 0, 1]) * (h / 6)
    return sp.csr_matrix((sp.kron(M1, K1) + sp.kron(K1, M1)) / h**2)


def fd3_matrix(n, h):
    import scipy.sparse as sp
    one = np.ones(n)
    A = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h**2
    I = sp.identity(n)
    return sp.csr_matrix(sp.kron(I, sp.kron(I, A)) + sp.kron(I, sp.kron(A, I))
                         + sp.kron(A, sp.kron(I, I)))


def subgrid_mask(n_side, per_axis, dim):
    stride = n_side // per_axis
    idx = stride // 2 + stride * np.arange(per_axis)
    mask = np.zeros(n_side ** dim, bool)
    if dim == 3:
        mask[(idx[:, None, None] * n_side**2 + idx[None, :, None] * n_side
              + idx[None, None, :]).ravel()] = True
    else:
        mask[(idx[:, None] * n_side + idx[None, :]).ravel()] = True
    return mask


def q1_prior_diag2(n_side, delta, gamma):
    """diag((δI + γ L_Q1)⁻²) through the separable DST-I eigenbasis of the
    Q1-lumped stiffness (SURVEY §8(c) eigenvalue formula); checked against a
    dense inverse at a small size before use."""
    h = 1.0 / (n_side + 1)
    m = np.arange(1, n_side + 1)
    c = np.cos(m * math.pi * h)
    k1, m1 = (2 / h) * (1 - c), (h / 3) * (2 + c)
    lam = (np.outer(m1, k1) + np.outer(k1, m1)) / h**2  # [m2, m1]
    i = np.arange(1, n_side + 1)
    phi = np.sqrt(2.0 / (n_side + 1)) * np.sin(np.outer(i, m) * math.pi * h)  # [i, m]
    d = (delta + gamma * lam) ** -2.0
    # diag_{i2, i1} = sum_{m2, m1} phi[i2,m2]^2 phi[i1,m1]^2 d[m2,m1]
    return ((phi ** 2) @ d @ (phi ** 2).T).ravel()  # row-major (i2, i1): x1 fastest


def _check_prior_diag():
    import scipy.sparse as sp
    n = 9
    h = 1.0 / (n + 1)
    A = (1.0 * sp.identity(n * n) + 0.05 * q1_matrix(n, h)).toarray()
    Pinv = np.linalg.inv(A)
    ref = np.diag(Pinv @ Pinv)
    got = q1_prior_diag2(n, 1.0, 0.05)
    assert np.allclose(got, ref, rtol=1e-12, atol=0), np.abs(got - ref).max()


class ConfigProblem:
    """The reference pipeline with a config operator/prior/time mask wrapped in."""

    def __init__(self, lp, hs, n_side, dim, L, n_t, mask, sigma, delta, gp, eps0, rmax,
                 every=1, mode="ic"):
        import scipy.sparse as sp
        import scipy.sparse.linalg as spla
        from lrpostcov.forward import DistributedInjection, InitInjection

        h = 1.0 / (n_side + 1)
        m = h ** dim
        n_x = n_side ** dim
        grid = SimpleNamespace(n_x=n_x, m_scale=m, n_side=n_side, h=h, d=dim)
        spatial = SimpleNamespace(grid=grid, L=L, m_scale=m, kind="heat")
        t0 = time.perf_counter()
        self.K = lp.SpaceTimeOperator(spatial, lp.build_time_grid(n_t))
        self.setup_s = time.perf_counter() - t0
        self.lp, self.hs = lp, hs
        self.layout = hs.SensorLayout(patches=(), mask=mask)
        tau = 1.0 / n_t
        self.beta_noise = 1.0 / (sigma ** 2 * tau * m)  # w = 1/σ²
        self.cov = hs.CovarianceSpec(beta_noise=self.beta_noise, beta_prior=1.0, gamma_prior=1.0)
        self.pol = lp.TruncationPolicy(eps0, rmax)
        self.P = spla.splu((delta * sp.identity(n_x) + gp * L).tocsc())
        self.every, self.n_t, self.n_x = every, n_t, n_x
        self.inj = InitInjection(self.K) if mode == "ic" else DistributedInjection(self.K)
        self.mode = mode
        self.rank_trace = []
        self.last = {}

    def _obs(self, Y):
        lp, hs = self.lp, self.hs
        Z = hs.apply_obs_weight(Y, self.layout, self.cov, self.K.time, self.K.m_scale, pol=None)
        if self.every > 1 and Z.r:
            keep = (np.arange(self.n_t) + 1) % self.every == 0
            Z = lp.LowRankMat(Z.W1, np.where(keep[:, None], Z.W2, 0.0))
        return lp.lr_truncate(Z, self.pol)

    def apply(self, v):
        """hessian.py:211-226 (IC) / :229-245 (source) with Γ^{1/2} = √γ P."""
        lp = self.lp
        sg = math.sqrt(self.cov.gamma_prior)
        fw, bw = [], []
        if self.mode == "ic":
            x = sg * self.P.solve(np.asarray(v, float))
            rhs = self.inj.rhs(x)
        else:
            rhs = self.inj.rhs(lp.LowRankMat(self.P.solve(v.W1), sg * v.W2))
        Y = lp.st_solve_sweep(self.K, rhs, self.pol, compress_every=4, trace=fw)
        Z = self._obs(Y)
        Q = lp.st_solve_adjoint_sweep(self.K, Z, self.pol, compress_every=4, trace=bw)
        local = fw + [Z.r] + bw
        if self.mode == "ic":
            out = sg * self.P.solve(self.inj.extract(Q))
        else:
            E = self.inj.extract(Q)
            out = lp.lr_truncate(lp.LowRankMat(self.P.solve(E.W1), sg * E.W2), self.pol)
            local.append(out.r)
        self.rank_trace.append(max(local))
        self.last = {"fwd": np.array(fw), "bwd": np.array(bw), "obs": Z.r}
        return out


def c2_problem(lp, hs):
    n = 256
    h = 1.0 / (n + 1)
    return ConfigProblem(lp, hs, n, 2, q1_matrix(n, h), 512, subgrid_mask(n, 32, 2), 0.01,
                         1.0, 0.05, 1e-8, 32)


def case_c2_apply(lp, hs):
    P = c2_problem(lp, hs)
    v = np.random.default_rng(1).standard_normal(P.n_x)
    v /= np.linalg.norm(v)
    t0 = time.perf_counter()
    O = P.apply(v)
    dt = time.perf_counter() - t0
    return {"O": O, "fwd": P.last["fwd"], "bwd": P.last["bwd"], "obs": np.array([P.last["obs"]]),
            "max_rank": np.array([P.rank_trace[-1]]), "seconds": np.array([dt, P.setup_s])}


def case_c2_arnoldi(lp, hs):
    from lrpostcov import posterior
    from lrpostcov.arnoldi import StopRule, lr_arnoldi

    _check_prior_diag()
    P = c2_problem(lp, hs)
    v1 = np.random.default_rng(1).standard_normal(P.n_x)
    v1 /= np.linalg.norm(v1)
    t0 = time.perf_counter()
    res = lr_arnoldi(P.apply, v1, P.pol, StopRule(m_a=50, eps_eig=1e-1, check_every=10),
                     rank_source=P.rank_trace)
    dt = time.perf_counter() - t0
    summ = posterior.build_summary(res.ritz_values, [np.asarray(v) for v in res.ritz_vectors],
                                   gamma_prior=1.0, eps_eig=1e-1, n_x=P.n_x)
    PV = np.column_stack([P.P.solve(summ.V[:, j]) for j in range(summ.k)]) if summ.k else \
        np.zeros((P.n_x, 0))
    reduction = (PV * PV) @ summ.filters
    var = q1_prior_diag2(256, 1.0, 0.05) - reduction
    return {"ritz": res.ritz_values.real, "ritz_imag": res.ritz_values.imag,
            "iters": np.array([res.iterations]), "H": res.H,
            "ranks": np.array(res.rank_trace), "retained": summ.eigenvalues,
            "var": var, "reduction": reduction, "seconds": np.array([dt])}


def case_c1_source(lp, hs):
    from lrpostcov.arnoldi import StopRule, lr_arnoldi
    from lrpostcov.lowrank import lr_singular_values

    n, n_t = 32, 64
    h = 1.0 / (n + 1)
    P = ConfigProblem(lp, hs, n, 2, q1_matrix(n, h), n_t, np.ones(n * n, bool), 0.01, 1.0, 0.1,
                      1e-8, 20, mode="source")
    rng = np.random.default_rng(0)  # cli.start_vector, source mode, start="random"
    w1 = rng.standard_normal((P.n_x, 1))
    w2 = rng.standard_normal((n_t, 1))
    w1 /= np.linalg.norm(w1)
    w2 /= np.linalg.norm(w2)
    v1 = lp.LowRankMat(w1, w2)
    t0 = time.perf_counter()
    res = lr_arnoldi(P.apply, v1, P.pol, StopRule(m_a=10, eps_eig=1e-1, check_every=10),
                     rank_source=P.rank_trace)
    dt = time.perf_counter() - t0
    top = res.ritz_vectors[0]
    return {"ritz": res.ritz_values.real, "ritz_imag": res.ritz_values.imag,
            "iters": np.array([res.iterations]), "H": res.H, "ranks": np.array(res.rank_trace),
            "basis_ranks": np.array([b.r for b in res.basis]),
            "top_sv": lr_singular_values(top),
            "w1": w1[:, 0], "w2": w2[:, 0], "seconds": np.array([dt])}


def case_c4_sweep3d(lp, hs):
    n, n_t = 48, 32
    h = 1.0 / (n + 1)
    P = ConfigProblem(lp, hs, n, 3, fd3_matrix(n, h), n_t, subgrid_mask(n, 12, 3), 0.005, 1.0,
                      0.02, 1e-8, 64, every=4)
    v = np.random.default_rng(3).standard_normal(P.n_x)
    v /= np.linalg.norm(v)
    t0 = time.perf_counter()
    O = P.apply(v)
    dt = time.perf_counter() - t0
    return {"O": O, "fwd": P.last["fwd"], "bwd": P.last["bwd"], "obs": np.array([P.last["obs"]]),
            "max_rank": np.array([P.rank_trace[-1]]), "seconds": np.array([dt, P.setup_s])}


def case_c1_gmres(lp, hs):
    """st_solve_krylov (forward.py:217-274) at the C1 operator size: Q1-lumped
    32², n_t 64, a seeded rank-2 rhs, eps0 1e-8, forward and adjoint."""
    n, n_t = 32, 64
    h = 1.0 / (n + 1)
    grid = SimpleNamespace(n_x=n * n, m_scale=h * h, n_side=n, h=h, d=2)
    spatial = SimpleNamespace(grid=grid, L=q1_matrix(n, h), m_scale=h * h, kind="heat")
    K = lp.SpaceTimeOperator(spatial, lp.build_time_grid(n_t))
    rng = np.random.default_rng(8)
    rhs = lp.lr_truncate(lp.LowRankMat(rng.standard_normal((n * n, 2)),
                                       rng.standard_normal((n_t, 2))), lp.TruncationPolicy())
    out = {"R1": rhs.W1, "R2": rhs.W2}
    for tag, adj in (("f", False), ("b", True)):
        tr = []
        t0 = time.perf_counter()
        Y = lp.st_solve_krylov(K, rhs, lp.TruncationPolicy(), adjoint=adj, trace=tr)
        out[f"{tag}_seconds"] = np.array([time.perf_counter() - t0])
        out[f"{tag}_Y1"], out[f"{tag}_Y2"] = Y.W1, Y.W2
        out[f"{tag}_trace"] = np.array(tr)
    return out


CASES = {"c1_gmres": case_c1_gmres, "c2_apply": case_c2_apply, "c2_arnoldi": case_c2_arnoldi,
         "c1_source": case_c1_source, "c4_sweep3d": case_c4_sweep3d}


def main(argv):
    sys.path.insert(0, REF)
    import lrpostcov as lp
    from lrpostcov import hessian as hs

    for name in (argv or list(CASES)):
        t0 = time.perf_counter()
        out = CASES[name](lp, hs)
        path = os.path.join(HERE, f"config_{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: {time.perf_counter() - t0:.1f} s -> {path} "
              f"({os.path.getsize(path) / 1e3:.0f} kB)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
