"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is mounted read-only there; it is
absent on the GPU box, so its outputs travel as these .npz files):

    python tests/golden/make_golden.py

Every case stores its seeded inputs and the reference's outputs.  The oracle
(oracle/lrk_oracle.py) is pinned against these files by
tests/test_oracle_golden.py, and the GPU parity tests reuse the same inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    import lrpostcov as lp
    from lrpostcov import hessian as hs

    out = {}

    # --- lr_truncate (lowrank.py:124-144) on decaying random spectra
    rng = np.random.default_rng(100)
    for name, (n, m, r, eps0, rmax) in {
        "trunc_a": (200, 150, 40, 1e-8, None),
        "trunc_b": (60, 200, 25, 1e-5, None),
        "trunc_c": (35, 35, 35, 1e-2, None),
        "trunc_d": (300, 64, 30, 1e-8, 7),
    }.items():
        W1 = rng.standard_normal((n, r)) * np.logspace(0, -9, r)
        W2 = rng.standard_normal((m, r))
        A = lp.lr_truncate(lp.LowRankMat(W1, W2), lp.TruncationPolicy(eps0, rmax))
        out[f"{name}_W1"], out[f"{name}_W2"] = W1, W2
        out[f"{name}_meta"] = np.array([eps0, -1 if rmax is None else rmax])
        out[f"{name}_U"], out[f"{name}_V"] = A.W1, A.W2

    # --- sweeps (forward.py:133-201)
    for name, (n_side, n_t, r, adjoint, seed) in {
        "sweep_a": (7, 5, 2, False, 1),
        "sweep_b": (15, 20, 3, False, 2),
        "sweep_c": (15, 21, 2, True, 3),
        "sweep_d": (31, 64, 1, False, 4),
    }.items():
        rng = np.random.default_rng(seed)
        grid = lp.build_grid(n_side)
        K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
        rhs = lp.lr_truncate(lp.LowRankMat(rng.standard_normal((grid.n_x, r)),
                                           rng.standard_normal((n_t, r))), lp.TruncationPolicy())
        tr = []
        Y = lp.st_solve_sweep(K, rhs, lp.TruncationPolicy(), adjoint=adjoint, trace=tr)
        out[f"{name}_meta"] = np.array([n_side, n_t, int(adjoint)])
        out[f"{name}_R1"], out[f"{name}_R2"] = rhs.W1, rhs.W2
        out[f"{name}_Y1"], out[f"{name}_Y2"] = Y.W1, Y.W2
        out[f"{name}_trace"] = np.array(tr)

    # --- GMRES on factored iterates (forward.py:217-274)
    rng = np.random.default_rng(8)
    grid = lp.build_grid(15)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(10))
    rhs = lp.lr_truncate(lp.LowRankMat(rng.standard_normal((grid.n_x, 2)),
                                       rng.standard_normal((10, 2))), lp.TruncationPolicy())
    tr = []
    Yk = lp.st_solve_krylov(K, rhs, lp.TruncationPolicy(), trace=tr)
    out["gmres_R1"], out["gmres_R2"] = rhs.W1, rhs.W2
    out["gmres_Y"] = lp.lr_to_dense(Yk)
    out["gmres_iters"] = np.array([len(tr)])

    # --- Hessian IC applies (hessian.py:211-226)
    for name, (n_side, n_t, layout_kind, gamma, ratio, seed, rmax) in {
        "hic_a": (7, 5, "full", 10.0, 1e4, 0, None),
        "hic_b": (15, 20, "3x3", 10.0, 1e4, 1, None),
        "hic_c": (31, 64, "sub8", 0.05, 1e6, 2, None),
        "hic_d": (32, 48, "sub8", 0.1, 1e5, 3, 6),
    }.items():
        grid = lp.build_grid(n_side)
        K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
        if layout_kind == "full":
            layout = hs.full_observation(grid)
        elif layout_kind == "3x3":
            layout = hs.make_sensor_layout_3x3(grid)
        else:
            stride = n_side // 8
            idx = stride // 2 + stride * np.arange(8)
            mask = np.zeros(grid.n_x, bool)
            mask[(idx[:, None] * n_side + idx[None, :]).ravel()] = True
            layout = hs.SensorLayout(patches=(), mask=mask)
        cov = hs.CovarianceSpec.from_gamma(gamma, ratio, grid)
        pol = lp.TruncationPolicy(1e-8, rmax)
        ctx = hs.HessianContext(mode=hs.MODE_IC, operator=K, layout=layout, cov=cov, pol=pol)
        V = np.random.default_rng(seed).standard_normal((grid.n_x, 3))
        V /= np.linalg.norm(V, axis=0)
        O = np.column_stack([ctx.apply(V[:, j]) for j in range(3)])
        out[f"{name}_meta"] = np.array([n_side, n_t, cov.beta_noise, cov.beta_prior,
                                        cov.gamma_prior, -1 if rmax is None else rmax])
        out[f"{name}_mask"] = layout.mask
        out[f"{name}_V"], out[f"{name}_O"] = V, O
        out[f"{name}_ranks"] = np.array(ctx.rank_trace)

    # --- Hessian source apply (hessian.py:229-245)
    grid = lp.build_grid(9)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(6))
    cov = hs.CovarianceSpec.from_gamma(10.0, 1e4, grid)
    ctx = hs.HessianContext(mode=hs.MODE_SOURCE, operator=K, layout=hs.full_observation(grid),
                            cov=cov, pol=lp.TruncationPolicy())
    rng = np.random.default_rng(5)
    v = lp.lr_truncate(lp.LowRankMat(rng.standard_normal((grid.n_x, 2)),
                                     rng.standard_normal((6, 2))), lp.TruncationPolicy())
    Hv = ctx.apply(v)
    out["hst_meta"] = np.array([9, 6, cov.beta_noise, cov.beta_prior, cov.gamma_prior])
    out["hst_V1"], out["hst_V2"] = v.W1, v.W2
    out["hst_O"] = lp.lr_to_dense(Hv)
    out["hst_ranks"] = np.array(ctx.rank_trace)

    # --- Arnoldi + posterior variance (arnoldi.py:271-375, posterior.py:65-111)
    from lrpostcov import posterior
    from lrpostcov.arnoldi import StopRule, lr_arnoldi

    grid = lp.build_grid(15)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(12))
    cov = hs.CovarianceSpec.from_gamma(1.0, 1e6, grid)
    ctx = hs.HessianContext(mode=hs.MODE_IC, operator=K, layout=hs.make_sensor_layout_3x3(grid),
                            cov=cov, pol=lp.TruncationPolicy())
    v1 = np.random.default_rng(7).standard_normal(grid.n_x)
    v1 /= np.linalg.norm(v1)
    res = lr_arnoldi(ctx.apply, v1, lp.TruncationPolicy(), StopRule(m_a=30, eps_eig=1e-1),
                     rank_source=ctx.rank_trace)
    summ = posterior.build_summary(res.ritz_values, res.ritz_vectors, cov.gamma_prior, 1e-1)
    out["arn_meta"] = np.array([15, 12, cov.beta_noise, cov.beta_prior, cov.gamma_prior, 30])
    out["arn_mask"] = ctx.layout.mask
    out["arn_v1"] = v1
    out["arn_ritz"] = res.ritz_values.real
    out["arn_iters"] = np.array([res.iterations])
    out["arn_var"] = summ.variance_field

    # --- convection-diffusion (the reference's own operator, discretize.py:115-127)
    for name, (n_side, n_t, nu, wind, adjoint, seed) in {
        "cdsw_a": (9, 8, 0.05, (1.0, -0.5), False, 31),
        "cdsw_b": (12, 10, 0.02, (-0.7, 1.3), True, 32),
    }.items():
        rng = np.random.default_rng(seed)
        grid = lp.build_grid(n_side)
        K = lp.SpaceTimeOperator(lp.assemble_convdiff(grid, nu, wind), lp.build_time_grid(n_t))
        rhs = lp.lr_truncate(lp.LowRankMat(rng.standard_normal((grid.n_x, 2)),
                                           rng.standard_normal((n_t, 2))), lp.TruncationPolicy())
        tr = []
        Y = lp.st_solve_sweep(K, rhs, lp.TruncationPolicy(), adjoint=adjoint, trace=tr)
        out[f"{name}_meta"] = np.array([n_side, n_t, int(adjoint), nu, wind[0], wind[1]])
        out[f"{name}_R1"], out[f"{name}_R2"] = rhs.W1, rhs.W2
        out[f"{name}_Y1"], out[f"{name}_Y2"] = Y.W1, Y.W2
        out[f"{name}_trace"] = np.array(tr)
    for name, (n_side, n_t, nu, wind, seed) in {
        "hcd_a": (15, 12, 0.05, (1.0, -0.5), 33),
        "hcd_b": (16, 16, 0.02, (0.4, 0.9), 34),
    }.items():
        grid = lp.build_grid(n_side)
        K = lp.SpaceTimeOperator(lp.assemble_convdiff(grid, nu, wind), lp.build_time_grid(n_t))
        stride = n_side // 4
        idx = stride // 2 + stride * np.arange(4)
        mask = np.zeros(grid.n_x, bool)
        mask[(idx[:, None] * n_side + idx[None, :]).ravel()] = True
        layout = hs.SensorLayout(patches=(), mask=mask)
        cov = hs.CovarianceSpec.from_gamma(1.0, 1e5, grid)
        ctx = hs.HessianContext(mode=hs.MODE_IC, operator=K, layout=layout, cov=cov,
                                pol=lp.TruncationPolicy(1e-8))
        V = np.random.default_rng(seed).standard_normal((grid.n_x, 2))
        V /= np.linalg.norm(V, axis=0)
        O = np.column_stack([ctx.apply(V[:, j]) for j in range(2)])
        out[f"{name}_meta"] = np.array([n_side, n_t, nu, wind[0], wind[1], cov.beta_noise,
                                        cov.beta_prior, cov.gamma_prior])
        out[f"{name}_mask"] = mask
        out[f"{name}_V"], out[f"{name}_O"] = V, O
        out[f"{name}_ranks"] = np.array(ctx.rank_trace)

    # --- config extensions: the UNMODIFIED reference pipeline
    # (st_solve_sweep / apply_obs_weight / lr_truncate / InitInjection) with the
    # config matrices duck-typed into SpaceTimeOperator, the (δI+γL)⁻¹ prior
    # wrapped around it and the time-row mask inserted before the truncation,
    # following hessian.py:211-226 line by line.
    import math

    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    from types import SimpleNamespace

    from lrpostcov.forward import InitInjection

    def q1_matrix(n, h):
        one = np.ones(n)
        K1 = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h
        M1 = sp.diags([one[1:], 4 * one, one[1:]], [-1, 0, 1]) * (h / 6)
        return sp.csr_matrix((sp.kron(M1, K1) + sp.kron(K1, M1)) / h**2)

    def fd3_matrix(n, h):
        one = np.ones(n)
        A = sp.diags([-one[1:], 2 * one, -one[1:]], [-1, 0, 1]) / h**2
        I = sp.identity(n)
        return sp.csr_matrix(sp.kron(I, sp.kron(I, A)) + sp.kron(I, sp.kron(A, I))
                             + sp.kron(A, sp.kron(I, I)))

    def rot_matrix(n, h, dim, nu, w0):
        # rotating-field convection diffusion; the assembly is the oracle's own
        # (test infrastructure): this fixture pins the reference pipeline run on it
        sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
        from oracle import lrk_oracle as O
        return O.config_operator(n, dim, "fd", "convdiff", nu, w0, "rotating")[0]

    s3 = 1.0 / math.sqrt(3.0)
    for name, (n_side, dim, stencil, n_t, sens, every, delta, gp, sigma, rmax, seed) in {
        "cfg_q1": (15, 2, "q1", 16, 5, 1, 1.0, 0.05, 0.01, None, 11),
        "cfg_q1b": (24, 2, "q1", 12, 8, 1, 1.0, 0.1, 0.01, 12, 12),
        "cfg_3d": (7, 3, "fd", 12, 3, 4, 1.0, 0.02, 0.005, None, 13),
        "cfg_rot": (14, 2, ("rot", 0.05, (0.0, 0.0, 0.0)), 12, 4, 1, 1.0, 0.05, 0.01, None, 14),
        "cfg_rot3": (6, 3, ("rot", 0.02, (s3, s3, s3)), 8, 3, 1, 1.0, 0.02, 0.005, None, 15),
    }.items():
        h = 1.0 / (n_side + 1)
        m = h ** dim
        if isinstance(stencil, tuple):
            L = rot_matrix(n_side, h, dim, stencil[1], stencil[2])
        else:
            L = q1_matrix(n_side, h) if stencil == "q1" else fd3_matrix(n_side, h)
        n_x = n_side ** dim
        grid = SimpleNamespace(n_x=n_x, m_scale=m, n_side=n_side, h=h, d=dim)
        spatial = SimpleNamespace(grid=grid, L=L, m_scale=m, kind="heat")
        K = lp.SpaceTimeOperator(spatial, lp.build_time_grid(n_t))
        stride = n_side // sens
        idx = stride // 2 + stride * np.arange(sens)
        mask = np.zeros(n_x, bool)
        if dim == 3:
            mask[(idx[:, None, None] * n_side**2 + idx[None, :, None] * n_side
                  + idx[None, None, :]).ravel()] = True
        else:
            mask[(idx[:, None] * n_side + idx[None, :]).ravel()] = True
        layout = hs.SensorLayout(patches=(), mask=mask)
        tau = 1.0 / n_t
        beta_noise = 1.0 / (sigma**2 * tau * m)  # w = 1/sigma^2
        cov = hs.CovarianceSpec(beta_noise=beta_noise, beta_prior=1.0, gamma_prior=1.0)
        pol = lp.TruncationPolicy(1e-8, rmax)
        Lprior = L if not isinstance(stencil, tuple) else \
            (fd3_matrix(n_side, h) if dim == 3 else lp.assemble_heat(lp.build_grid(n_side)).L)
        P = spla.splu((delta * sp.identity(n_x) + gp * Lprior).tocsc())
        inj = InitInjection(K)

        def apply(v):
            local = []
            x = math.sqrt(cov.gamma_prior) * P.solve(v)
            Y = lp.st_solve_sweep(K, inj.rhs(x), pol, compress_every=4, trace=local)
            Z = hs.apply_obs_weight(Y, layout, cov, K.time, K.m_scale, pol=None)
            if every > 1 and Z.r:
                keep = (np.arange(n_t) + 1) % every == 0
                Z = lp.LowRankMat(Z.W1, np.where(keep[:, None], Z.W2, 0.0))
            Z = lp.lr_truncate(Z, pol)
            local.append(Z.r)
            Q = lp.st_solve_adjoint_sweep(K, Z, pol, compress_every=4, trace=local)
            return math.sqrt(cov.gamma_prior) * P.solve(inj.extract(Q)), max(local)

        V = np.random.default_rng(seed).standard_normal((n_x, 2))
        V /= np.linalg.norm(V, axis=0)
        res = [apply(V[:, j]) for j in range(2)]
        kind_code = 2 if isinstance(stencil, tuple) else (1 if stencil == "q1" else 0)
        nu_w = stencil[1:] if isinstance(stencil, tuple) else (0.0, (0.0, 0.0, 0.0))
        out[f"{name}_meta"] = np.array([n_side, dim, kind_code, n_t, every, delta, gp, beta_noise,
                                        -1 if rmax is None else rmax, nu_w[0], *nu_w[1]])
        out[f"{name}_mask"] = mask
        out[f"{name}_V"] = V
        out[f"{name}_O"] = np.column_stack([r[0] for r in res])
        out[f"{name}_ranks"] = np.array([r[1] for r in res])

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
