"""Pin the CPU oracle against the reference's own outputs (tests/golden) and
the reference's closed-form known answers.  CPU only."""


import numpy as np
import pytest

from oracle import lrk_oracle as O


def _rmax(v):
    return None if v < 0 else int(v)


@pytest.mark.parametrize("name", ["trunc_a", "trunc_b", "trunc_c", "trunc_d"])
def test_truncate_matches_reference(golden, name):
    eps0, rmax = golden[f"{name}_meta"]
    U, V = O.truncate(golden[f"{name}_W1"], golden[f"{name}_W2"], eps0, _rmax(rmax))
    assert U.shape == golden[f"{name}_U"].shape
    np.testing.assert_allclose(U, golden[f"{name}_U"], atol=1e-12)
    np.testing.assert_allclose(V, golden[f"{name}_V"], rtol=1e-12, atol=1e-12 * np.abs(V).max())


@pytest.mark.parametrize("name", ["sweep_a", "sweep_b", "sweep_c", "sweep_d"])
def test_sweep_matches_reference(golden, name):
    n_side, n_t, adjoint = (int(x) for x in golden[f"{name}_meta"])
    L, h, m = O.fd_operator(n_side)
    solver = O.StepSolver(L, m, 1.0 / n_t, n_t)
    Y1, Y2, tr = O.sweep(solver, golden[f"{name}_R1"], golden[f"{name}_R2"], 1e-8, None,
                         bool(adjoint))
    assert tr == golden[f"{name}_trace"].tolist()
    ref = golden[f"{name}_Y1"] @ golden[f"{name}_Y2"].T
    assert np.linalg.norm(Y1 @ Y2.T - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("name", ["cdsw_a", "cdsw_b"])
def test_convdiff_sweep_matches_reference(golden, name):
    n_side, n_t, adjoint, nu, w1, w2 = golden[f"{name}_meta"]
    L, h, m = O.fd_operator(int(n_side), "convdiff", nu, (w1, w2))
    solver = O.StepSolver(L, m, 1.0 / n_t, int(n_t))
    Y1, Y2, tr = O.sweep(solver, golden[f"{name}_R1"], golden[f"{name}_R2"], 1e-8, None,
                         bool(adjoint))
    assert tr == golden[f"{name}_trace"].tolist()
    ref = golden[f"{name}_Y1"] @ golden[f"{name}_Y2"].T
    assert np.linalg.norm(Y1 @ Y2.T - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("name", ["hcd_a", "hcd_b"])
def test_convdiff_hessian_ic_matches_reference(golden, name):
    n_side, n_t, nu, w1, w2, bn, bp, g = golden[f"{name}_meta"]
    P = O.Problem(int(n_side), int(n_t), golden[f"{name}_mask"], bn, g, 1e-8, kind="convdiff",
                  nu=nu, wind=(w1, w2))
    V, Oref = golden[f"{name}_V"], golden[f"{name}_O"]
    ranks = []
    for j in range(V.shape[1]):
        out, r = O.hessian_ic(P, V[:, j])
        ranks.append(r)
        assert np.linalg.norm(out - Oref[:, j]) <= 1e-12 * np.linalg.norm(Oref[:, j])
    assert ranks == golden[f"{name}_ranks"].tolist()


def test_gmres_matches_reference(golden):
    L, h, m = O.fd_operator(15)
    solver = O.StepSolver(L, m, 0.1, 10)
    (Y1, Y2), iters, tr = O.gmres(solver, golden["gmres_R1"], golden["gmres_R2"], 1e-8)
    assert iters == int(golden["gmres_iters"][0])
    ref = golden["gmres_Y"]
    assert np.linalg.norm(Y1 @ Y2.T - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("name", ["hic_a", "hic_b", "hic_c", "hic_d"])
def test_hessian_ic_matches_reference(golden, name):
    n_side, n_t, bn, bp, g, rmax = golden[f"{name}_meta"]
    P = O.Problem(int(n_side), int(n_t), golden[f"{name}_mask"], bn, g, 1e-8, _rmax(rmax))
    V, Oref = golden[f"{name}_V"], golden[f"{name}_O"]
    ranks = []
    for j in range(V.shape[1]):
        out, r = O.hessian_ic(P, V[:, j])
        ranks.append(r)
        assert np.linalg.norm(out - Oref[:, j]) <= 1e-12 * np.linalg.norm(Oref[:, j])
    assert ranks == golden[f"{name}_ranks"].tolist()


CFG = ["cfg_q1", "cfg_q1b", "cfg_3d", "cfg_rot", "cfg_rot3"]


def cfg_problem(golden, name):
    n_side, dim, code, n_t, every, delta, gp, bn, rmax, nu, w0, w1, w2 = golden[f"{name}_meta"]
    extra = dict(kind="convdiff", nu=nu, wind=(w0, w1, w2), wind_field="rotating") if code == 2 else {}
    return O.Problem(int(n_side), int(n_t), golden[f"{name}_mask"], bn, 1.0, 1e-8, _rmax(rmax),
                     dim=int(dim), stencil="q1" if code == 1 else "fd", prior=(delta, gp),
                     obs_every=int(every), **extra)


@pytest.mark.parametrize("name", CFG)
def test_config_hessian_ic_matches_reference(golden, name):
    """Config extensions (Q1-lumped, 3-D 7-point, (δI+γL)⁻¹ prior, time-subsampled
    sensors) against the unmodified reference pipeline run with the same
    matrices duck-typed in (tests/golden/make_golden.py)."""
    P = cfg_problem(golden, name)
    V, Oref = golden[f"{name}_V"], golden[f"{name}_O"]
    ranks = []
    for j in range(V.shape[1]):
        out, r = O.hessian_ic(P, V[:, j])
        ranks.append(r)
        assert np.linalg.norm(out - Oref[:, j]) <= 1e-12 * np.linalg.norm(Oref[:, j])
    assert ranks == golden[f"{name}_ranks"].tolist()


@pytest.mark.parametrize("dim,stencil,modes,every", [
    (2, "q1", (1, 1), 1), (2, "q1", (3, 5), 1), (2, "q1", (7, 2), 4),
    (3, "fd", (1, 1, 1), 1), (3, "fd", (2, 1, 3), 4),
])
def test_config_full_observation_closed_form(dim, stencil, modes, every):
    """μ = β τ M Σ_{k observed} θ^{2k} (δ+γλ)⁻² on DST-I modes."""
    n_side, n_t, bn, prior = (12 if dim == 2 else 6), 16, 1e4, (1.0, 0.05)
    P = O.Problem(n_side, n_t, np.ones(n_side ** dim, bool), bn, 1.0, 1e-10, dim=dim,
                  stencil=stencil, prior=prior, obs_every=every)
    v = O.config_eigvec(modes, n_side)
    out, _ = O.hessian_ic(P, v)
    mu = O.config_ic_eigenvalue(modes, n_side, n_t, bn, 1.0, stencil, prior, every)
    assert np.linalg.norm(out - mu * v) <= 1e-9 * mu


def test_hessian_source_matches_reference(golden):
    n_side, n_t, bn, bp, g = golden["hst_meta"]
    P = O.Problem(int(n_side), int(n_t), np.ones(int(n_side) ** 2, bool), bn, g)
    (W1, W2), r = O.hessian_st(P, golden["hst_V1"], golden["hst_V2"])
    ref = golden["hst_O"]
    assert np.linalg.norm(W1 @ W2.T - ref) <= 1e-12 * np.linalg.norm(ref)
    assert r == int(golden["hst_ranks"][0])


def test_arnoldi_and_variance_match_reference(golden):
    n_side, n_t, bn, bp, g, m_a = golden["arn_meta"]
    P = O.Problem(int(n_side), int(n_t), golden["arn_mask"], bn, g)
    H, basis, vals, iters = O.arnoldi_dense(lambda x: O.hessian_ic(P, x)[0], golden["arn_v1"],
                                            int(m_a))
    assert iters == int(golden["arn_iters"][0])
    ref = golden["arn_ritz"]
    lead = ref >= 1e-1
    np.testing.assert_allclose(vals.real[lead], ref[lead], rtol=1e-10)
    rv, vecs = O.ritz_vectors(H, basis)
    var = O.posterior_variance(rv, vecs, g, 1e-1)
    np.testing.assert_allclose(var, golden["arn_var"], rtol=1e-10)


# ---- closed-form known answers used by the reference's own tests
def test_eigvec_injection_geometric_decay():
    """test_forward.py:40-48: y_k = θ^k v for an FD eigenvector."""
    n_side, n_t = 7, 5
    L, h, m = O.fd_operator(n_side)
    solver = O.StepSolver(L, m, 1.0 / n_t, n_t)
    v = O.fd_eigvec(1, 1, n_side)
    e0 = np.zeros((n_t, 1)); e0[0] = 1
    Y1, Y2, _ = O.sweep(solver, (m * v)[:, None], e0, 1e-8)
    theta = 1.0 / (1.0 + O.fd_eig(1, 1, n_side) / n_t)
    expect = np.column_stack([theta ** k * v for k in range(1, n_t + 1)])
    assert np.abs(Y1 @ Y2.T - expect).max() <= 1e-10


@pytest.mark.parametrize("m,n", [(1, 1), (2, 1), (3, 3)])
def test_full_observation_ic_eigenvalue(m, n):
    """test_hessian.py:129-139: μ = γ β τ M Σ θ^{2k}."""
    n_side, n_t = 7, 5
    h = 1.0 / (n_side + 1)
    gamma, ratio = 10.0, 1e4
    beta_prior = 1.0 / (gamma * h * h)
    P = O.Problem(n_side, n_t, np.ones(n_side ** 2, bool), ratio * beta_prior, gamma)
    v = O.fd_eigvec(m, n, n_side)
    out, _ = O.hessian_ic(P, v)
    mu = O.ic_eigenvalue_full_obs(m, n, n_side, n_t, ratio * beta_prior, gamma)
    assert np.linalg.norm(out - mu * v) <= 1e-8 * mu


def test_rank_cut_semantics():
    assert O.rank_cut(np.array([1.0, 1e-12]), 1e-8) == 1
    assert O.rank_cut(np.array([1.0, 0.5, 0.1]), 1e-8, r_max=2) == 2
    assert O.rank_cut(np.zeros(3), 1e-8) == 0
    assert O.rank_cut(np.array([1.0, 1e-16]), 1e-20) == 1  # noise floor


def test_galerkin_q1_convection_assembly():
    """Config C3 operator (extension): the product's
    vectorised closed-form element matrices, the oracle's Gauss-quadrature
    assembly, and (constant wind) the Kronecker closed form
    N = w1 M1 (x) C1 + w2 C1 (x) M1 agree."""
    import scipy.sparse as sp

    import paper_1703_05638_b200 as lp

    n = 7
    g = lp.build_grid(n)
    for field, w in (("const", (0.7, -1.3)), ("rotating", (0.0, 0.0)), ("rotating", (0.3, 0.2))):
        A = lp.assemble_convdiff(g, 0.05, w, field=field, scheme="galerkin").L
        B, h, m = O.config_operator(n, 2, "q1", "convdiff", 0.05, w, field)
        assert abs(A - B).max() < 1e-13 * abs(A).max()
        assert m == h * h
    h, one, w = g.h, np.ones(n), (0.7, -1.3)
    C1 = sp.diags([-one[1:], one[1:]], [-1, 1]) * 0.5
    M1 = sp.diags([one[1:], 4 * one, one[1:]], [-1, 0, 1]) * (h / 6)
    N = (w[0] * sp.kron(M1, C1) + w[1] * sp.kron(C1, M1)) / h**2
    A = lp.assemble_convdiff(g, 0.05, w, scheme="galerkin").L - 0.05 * lp.assemble_heat(g, "q1").L
    assert abs(A - N).max() < 1e-13 * abs(N).max()
    # element Peclet number of config C3 (nu = 1/20, n_side 512, |w| <= 2): SUPG inactive
    assert 2.0 * (1.0 / 513) / (2 * (1 / 20)) < 1.0
