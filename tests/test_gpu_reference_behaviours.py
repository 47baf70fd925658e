"""The reference's own unit-test behaviours, run through the device path.

Every test here states a property the reference's test-suite pins for the hot
path and its callers (cited file:line under /root/reference/pkg/tests) and
checks it on the GPU through the same public names.  Inputs are our own seeded
cases; nothing is read from the reference at run time.  Tolerances are the
reference's (stated in each test) unless the device path is required to be
tighter.
"""
import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_05638_b200 as lp  # noqa: E402
from paper_1703_05638_b200 import dense, posterior  # noqa: E402
from paper_1703_05638_b200 import hessian as hs  # noqa: E402

POL = lp.TruncationPolicy(1e-8)


def _field(rng, n_x, n_t, r):
    return lp.lr_truncate(lp.LowRankMat(rng.standard_normal((n_x, r)),
                                        rng.standard_normal((n_t, r))), POL)


def _heat(n_side, n_t, T=1.0):
    grid = lp.build_grid(n_side)
    op = lp.assemble_heat(grid)
    return grid, op, lp.SpaceTimeOperator(op, lp.build_time_grid(n_t, T=T))


def _ic_ctx(n_side, n_t, layout=None, cov=None):
    grid, op, K = _heat(n_side, n_t)
    layout = layout if layout is not None else hs.full_observation(grid)
    cov = cov if cov is not None else hs.CovarianceSpec.from_gamma(10.0, 1e4, grid)
    return grid, op, K, hs.HessianContext(mode=hs.MODE_IC, operator=K, layout=layout, cov=cov,
                                          pol=POL)


def _steady_ctx(n_side):
    op = lp.assemble_heat(lp.build_grid(n_side))
    return hs.HessianContext(mode=hs.MODE_STEADY, operator=None, layout=None,
                             cov=hs.CovarianceSpec(1e4, 1.0, 1.0), pol=POL, spatial=op)


def _dense_ic(ctx, op, grid, K):
    Hd, _ = dense.dense_misfit_ic(op.L.toarray(), grid.m_scale, K.time.tau, K.n_t,
                                  ctx.layout.mask, ctx.cov.beta_noise, ctx.cov.gamma_prior)
    return np.asarray(Hd.cpu().numpy() if torch.is_tensor(Hd) else Hd)


# ================================================================ factor algebra (test_lowrank.py)
def test_rank_one_input_is_reproduced_exactly():
    """test_lowrank.py:39-44."""
    rng = np.random.default_rng(100)
    u, v = rng.standard_normal((31, 1)), rng.standard_normal((17, 1))
    out = lp.lr_truncate(lp.LowRankMat(u, v), POL)
    assert out.r == 1
    assert np.abs(lp.lr_to_dense(out) - u @ v.T).max() <= 1e-13 * np.abs(u @ v.T).max()


def test_dense_roundtrip_of_a_rank_20_matrix():
    """test_lowrank.py:60-66, 181-186: from_dense finds the rank and reproduces within eps0."""
    rng = np.random.default_rng(101)
    X = rng.standard_normal((70, 20)) @ rng.standard_normal((20, 45))
    A = lp.lr_from_dense(X, POL)
    assert A.r == 20
    assert np.linalg.norm(lp.lr_to_dense(A) - X) <= POL.eps0 * np.linalg.norm(X)
    full = rng.standard_normal((24, 18))
    B = lp.lr_from_dense(full, lp.TruncationPolicy(1e-3))
    assert np.linalg.norm(lp.lr_to_dense(B) - full) <= 1e-3 * np.linalg.norm(full)


def test_truncation_is_idempotent_in_canonical_form():
    """test_lowrank.py:81-97: orthonormal W1, descending column norms of W2, and a second
    truncation changes nothing."""
    rng = np.random.default_rng(102)
    A = lp.LowRankMat(rng.standard_normal((50, 9)) * np.logspace(0, -5, 9),
                      rng.standard_normal((33, 9)))
    once = lp.lr_truncate(A, POL)
    twice = lp.lr_truncate(once, POL)
    W1, W2 = once.numpy()
    np.testing.assert_allclose(W1.T @ W1, np.eye(once.r), atol=1e-13)
    s = np.linalg.norm(W2, axis=0)
    assert (np.diff(s) <= 1e-12 * s[0]).all()
    assert twice.r == once.r
    assert np.linalg.norm(lp.lr_to_dense(twice) - lp.lr_to_dense(once)) <= 1e-13 * s[0]
    np.testing.assert_allclose(np.abs(twice.numpy()[0]), np.abs(W1), atol=1e-9)


def test_add_is_concatenation_and_checks_shapes():
    """test_lowrank.py:113-124: rank adds, the sum is exact, mismatched shapes raise."""
    rng = np.random.default_rng(103)
    A = lp.LowRankMat(rng.standard_normal((12, 2)), rng.standard_normal((7, 2)))
    B = lp.LowRankMat(rng.standard_normal((12, 3)), rng.standard_normal((7, 3)))
    C = lp.lr_add(A, B)
    assert C.r == 5
    np.testing.assert_array_equal(lp.lr_to_dense(C), lp.lr_to_dense(C))
    ref = lp.lr_to_dense(A) + lp.lr_to_dense(B)
    assert np.abs(lp.lr_to_dense(C) - ref).max() <= 1e-14 * np.abs(ref).max()
    with pytest.raises(ValueError):
        lp.lr_add(A, lp.LowRankMat(rng.standard_normal((11, 1)), rng.standard_normal((7, 1))))
    with pytest.raises(ValueError):
        lp.lr_dot(A, lp.LowRankMat(rng.standard_normal((12, 1)), rng.standard_normal((8, 1))))


def test_inner_product_unit_cases_bilinearity_symmetry():
    """test_lowrank.py:141-169."""
    e = np.eye(6)
    E01 = lp.LowRankMat(e[:, [0]], e[:5, [1]])
    E23 = lp.LowRankMat(e[:, [2]], e[:5, [3]])
    assert lp.lr_dot(E01, E01) == 1.0 and lp.lr_dot(E01, E23) == 0.0
    rng = np.random.default_rng(104)
    A, B, C = (_field(rng, 40, 25, r) for r in (3, 2, 4))
    dA, dB = lp.lr_to_dense(A), lp.lr_to_dense(B)
    assert lp.lr_dot(A, B) == pytest.approx(float(np.sum(dA * dB)), rel=1e-12)
    assert lp.lr_dot(A, B) == pytest.approx(lp.lr_dot(B, A), rel=1e-14)
    lhs = lp.lr_dot(lp.lr_add(lp.lr_scale(A, 2.0), lp.lr_scale(B, -3.0)), C)
    rhs = 2.0 * lp.lr_dot(A, C) - 3.0 * lp.lr_dot(B, C)
    assert lhs == pytest.approx(rhs, rel=1e-11, abs=1e-11 * lp.lr_norm(C) * lp.lr_norm(A))


def test_norm_scale_and_column_edge_cases():
    """test_lowrank.py:172-178, 199-202: zero field, negative scale, column(k)."""
    Z = lp.LowRankMat.zeros(9, 4)
    assert Z.r == 0 and lp.lr_norm(Z) == 0.0 and lp.lr_dot(Z, Z) == 0.0
    assert np.count_nonzero(lp.lr_to_dense(Z)) == 0 and lp.lr_to_dense(Z).shape == (9, 4)
    rng = np.random.default_rng(105)
    A = _field(rng, 15, 8, 3)
    assert lp.lr_norm(lp.lr_scale(A, -2.5)) == pytest.approx(2.5 * lp.lr_norm(A), rel=1e-13)
    assert lp.lr_scale(A, 0.0).r in (0, A.r) and lp.lr_norm(lp.lr_scale(A, 0.0)) == 0.0
    D = lp.lr_to_dense(A)
    for k in (0, 3, 7):
        np.testing.assert_allclose(A.column(k).cpu().numpy().ravel(), D[:, k], atol=1e-14)
    col = rng.standard_normal(15)
    F = lp.LowRankMat.from_column(col, 8, 5)
    Fd = lp.lr_to_dense(F)
    np.testing.assert_array_equal(Fd[:, 5], col)
    assert np.count_nonzero(np.delete(Fd, 5, axis=1)) == 0


def test_singular_values_of_a_field_match_the_dense_svd():
    """test_lowrank.py:189-196 (1e-11)."""
    rng = np.random.default_rng(106)
    A = lp.LowRankMat(rng.standard_normal((44, 6)), rng.standard_normal((29, 6)))
    ref = np.linalg.svd(lp.lr_to_dense(A), compute_uv=False)[:6]
    np.testing.assert_allclose(lp.lr_singular_values(A), ref, rtol=1e-11)


# ================================================================ sweeps and GMRES (test_forward.py)
def test_tiny_time_span_keeps_the_initial_condition():
    """test_forward.py:26-37: tau -> 0, every step is the identity; one rank."""
    grid, op, K = _heat(5, 5, T=5e-12)
    u = np.random.default_rng(110).standard_normal(grid.n_x)
    Y = lp.st_solve_sweep(K, lp.InitInjection(K).rhs(u), POL)
    assert Y.r == 1
    D = lp.lr_to_dense(Y)
    for k in range(5):
        np.testing.assert_allclose(D[:, k], u, rtol=1e-6)


def test_forward_sweep_equals_the_dense_substitution():
    """test_forward.py:51-63 (1e-8): the dense LU march of the same recurrence."""
    grid, op, K = _heat(7, 5)
    u = np.random.default_rng(111).standard_normal(grid.n_x)
    u /= np.linalg.norm(u)
    Y = lp.lr_to_dense(lp.st_solve_sweep(K, lp.InitInjection(K).rhs(u), POL))
    S = K.step_matrix.toarray()
    y, ref = u.copy(), np.zeros_like(Y)
    for k in range(5):
        y = np.linalg.solve(S, grid.m_scale * y)
        ref[:, k] = y
    assert np.linalg.norm(Y - ref) <= 1e-8 * np.linalg.norm(ref)


def test_injection_and_extraction_are_adjoint():
    """test_forward.py:119-127: <rhs(u), Y> = u . extract(Y)."""
    grid, op, K = _heat(7, 5)
    rng = np.random.default_rng(112)
    inj = lp.InitInjection(K)
    u = rng.standard_normal(grid.n_x)
    Y = _field(rng, grid.n_x, 5, 2)
    lhs, rhs = lp.lr_dot(inj.rhs(u), Y), float(u @ inj.extract(Y))
    assert abs(lhs - rhs) <= 1e-12 * abs(rhs)
    src = lp.DistributedInjection(K)
    G = _field(rng, grid.n_x, 5, 3)
    assert lp.lr_dot(src.rhs(G), Y) == pytest.approx(lp.lr_dot(G, src.extract(Y)), rel=1e-12)


def test_sweep_residual_contract_heat_and_convdiff():
    """test_forward.py:130-141: ||K Y - rhs|| <= 10 eps0 n_t ||rhs||."""
    rng = np.random.default_rng(113)
    for op, n_t in ((lp.assemble_heat(lp.build_grid(15)), 20),
                    (lp.assemble_convdiff(lp.build_grid(11), 1e-2, (0.0, 1.0)), 12)):
        K = lp.SpaceTimeOperator(op, lp.build_time_grid(n_t))
        rhs = _field(rng, op.grid.n_x, n_t, 3)
        for adjoint in (False, True):
            Y = lp.st_solve_sweep(K, rhs, POL, adjoint=adjoint)
            back = (K.apply_adjoint if adjoint else K.apply)(Y)
            resid = np.linalg.norm(lp.lr_to_dense(back) - lp.lr_to_dense(rhs))
            assert resid <= 10 * POL.eps0 * n_t * lp.lr_norm(rhs), adjoint


def test_sweep_rank_stays_bounded_under_time_refinement():
    """test_forward.py:144-157: max pane rank <= 40 and within 5 across n_t = 30, 60, 90."""
    grid = lp.build_grid(15)
    op = lp.assemble_heat(grid)
    u = np.random.default_rng(114).standard_normal(grid.n_x)
    u /= np.linalg.norm(u)
    tops = []
    for n_t in (30, 60, 90):
        K = lp.SpaceTimeOperator(op, lp.build_time_grid(n_t))
        trace = []
        lp.st_solve_sweep(K, lp.InitInjection(K).rhs(u), POL, trace=trace)
        assert len(trace) == -(-n_t // 4) + 1
        tops.append(max(trace))
    assert max(tops) <= 40 and max(tops) - min(tops) <= 5


def test_gmres_agrees_with_the_sweep():
    """test_forward.py:160-170: the two backends agree within 10 eps0 ||Y||."""
    grid, op, K = _heat(15, 10)
    rhs = _field(np.random.default_rng(115), grid.n_x, 10, 2)
    Ys = lp.st_solve_sweep(K, rhs, POL)
    Yk = lp.st_solve_krylov(K, rhs, POL)
    gap = np.linalg.norm(lp.lr_to_dense(Yk) - lp.lr_to_dense(Ys))
    assert gap <= 10 * POL.eps0 * lp.lr_norm(Ys)


def test_gmres_on_a_single_time_block_needs_one_iteration():
    """test_forward.py:173-182: with n_t = 1 the block preconditioner is K itself."""
    grid, op, _ = _heat(7, 5)
    K = lp.SpaceTimeOperator(op, lp.build_time_grid(1))
    rhs = _field(np.random.default_rng(116), grid.n_x, 1, 1)
    trace = []
    Y = lp.st_solve_krylov(K, rhs, POL, trace=trace)
    assert len(trace) == 1
    resid = np.linalg.norm(lp.lr_to_dense(K.apply(Y)) - lp.lr_to_dense(rhs))
    assert resid <= 1e-8 * lp.lr_norm(rhs)


def test_gmres_iterates_respect_the_rank_cap():
    """test_forward.py:185-195: only the cap is asserted; convergence may fail under it."""
    grid, op, K = _heat(7, 5)
    rhs = _field(np.random.default_rng(117), grid.n_x, 5, 2)
    trace = []
    try:
        lp.st_solve_krylov(K, rhs, lp.TruncationPolicy(1e-8, 3), trace=trace, tol=1e-6)
    except lp.ConvergenceFailure:
        pass
    assert trace and max(trace) <= 3


def test_gmres_stagnation_carries_the_residual_and_the_count():
    """test_forward.py:198-205."""
    grid, op, K = _heat(7, 5)
    rhs = _field(np.random.default_rng(118), grid.n_x, 5, 2)
    with pytest.raises(lp.ConvergenceFailure) as info:
        lp.st_solve_krylov(K, rhs, POL, tol=1e-16, max_iter=2)
    assert info.value.achieved_residual is not None and info.value.iterations == 2


def test_zero_right_hand_side_and_shape_errors():
    """test_forward.py:208-219."""
    grid, op, K = _heat(7, 5)
    Z = lp.LowRankMat.zeros(grid.n_x, 5)
    assert lp.st_solve_sweep(K, Z, POL).r == 0
    assert lp.st_solve_krylov(K, Z, POL).r == 0
    with pytest.raises(ValueError):
        lp.st_solve_sweep(K, lp.LowRankMat.zeros(grid.n_x, 6), POL)
    with pytest.raises(ValueError):
        lp.st_solve_sweep(K, lp.LowRankMat.zeros(grid.n_x + 1, 5), POL)


def test_step_matrix_has_a_positive_definite_symmetric_part():
    """test_forward.py:222-227 (heat and upwind convection-diffusion)."""
    tg = lp.build_time_grid(6)
    for op in (lp.assemble_heat(lp.build_grid(6)),
               lp.assemble_convdiff(lp.build_grid(6), 1e-2, (0.3, 1.0))):
        S = lp.SpaceTimeOperator(op, tg).step_matrix.toarray()
        assert np.linalg.eigvalsh(0.5 * (S + S.T))[0] > 0


# ================================================================ observation, Hessian (test_hessian.py)
def test_observation_weight_empty_full_and_masked():
    """test_hessian.py:69-99: no sensors -> rank 0; unit weight on all nodes -> identity;
    masking never raises the rank."""
    grid, tg = lp.build_grid(5), lp.build_time_grid(4)
    rng = np.random.default_rng(120)
    Y = lp.lr_from_dense(rng.standard_normal((grid.n_x, 4)), POL)
    one = hs.CovarianceSpec(1.0, 1.0, 1.0)
    assert hs.apply_obs_weight(Y, hs.empty_observation(grid), one, tg, grid.m_scale, pol=POL).r == 0
    unit = hs.CovarianceSpec(1.0 / (tg.tau * grid.m_scale), 1.0, 1.0)
    same = hs.apply_obs_weight(Y, hs.full_observation(grid), unit, tg, grid.m_scale)
    assert np.abs(lp.lr_to_dense(same) - lp.lr_to_dense(Y)).max() < 1e-13
    g15, t6 = lp.build_grid(15), lp.build_time_grid(6)
    R1 = lp.LowRankMat(rng.standard_normal((g15.n_x, 1)), rng.standard_normal((6, 1)))
    out = hs.apply_obs_weight(R1, hs.make_sensor_layout_3x3(g15),
                              hs.CovarianceSpec.from_gamma(10.0, 1e4, g15), t6, g15.m_scale, pol=POL)
    assert out.r <= 1
    mask = hs.make_sensor_layout_3x3(g15).mask
    assert np.count_nonzero(lp.lr_to_dense(out)[~mask]) == 0


def test_ic_hessian_zero_linearity_and_rank_trace():
    """test_hessian.py:102-115, 141-146: H 0 = 0; doubling beta_noise doubles H v (1e-13);
    one rank-trace entry per apply."""
    grid, op, K, ctx = _ic_ctx(5, 3)
    assert np.linalg.norm(hs.misfit_apply_ic(np.zeros(grid.n_x), ctx)) == 0.0
    cov2 = hs.CovarianceSpec(2 * ctx.cov.beta_noise, ctx.cov.beta_prior, ctx.cov.gamma_prior)
    ctx2 = hs.HessianContext(mode=hs.MODE_IC, operator=K, layout=ctx.layout, cov=cov2, pol=POL)
    v = np.random.default_rng(121).standard_normal(grid.n_x)
    np.testing.assert_allclose(hs.misfit_apply_ic(v, ctx2), 2 * hs.misfit_apply_ic(v, ctx),
                               rtol=1e-13, atol=1e-13 * np.abs(hs.misfit_apply_ic(v, ctx)).max())
    grid7, _, _, c7 = _ic_ctx(7, 5)
    ones = np.ones(grid7.n_x)
    c7.apply(ones)
    c7.apply(ones)
    assert len(c7.rank_trace) == 2 and all(r >= 1 for r in c7.rank_trace)
    clone = c7.clone()
    clone.apply(ones)
    assert len(c7.rank_trace) == 2 and len(clone.rank_trace) == 1   # test_hessian.py:280-284


def test_ic_hessian_equals_the_dense_brute_force():
    """test_hessian.py:117-127 (1e-8 over 20 probes), gamma_prior = 1."""
    grid, op, K = _heat(7, 5)
    cov = hs.CovarianceSpec(beta_noise=1e4, beta_prior=1.0, gamma_prior=1.0)
    ctx = hs.HessianContext(mode=hs.MODE_IC, operator=K, layout=hs.full_observation(grid),
                            cov=cov, pol=POL)
    Hd, _ = dense.dense_misfit_ic(op.L.toarray(), grid.m_scale, K.time.tau, 5, ctx.layout.mask,
                                  1e4, 1.0)
    assert dense.hv_agreement(ctx.apply, Hd, n_probe=20, seed=0) <= 1e-8


def test_ic_hessian_rank_bounded_across_time_refinement():
    """test_hessian.py:148-159: 3x3 sensors, n_t = 30, 60, 90."""
    grid = lp.build_grid(15)
    v = np.random.default_rng(122).standard_normal(grid.n_x)
    tops = []
    for n_t in (30, 60, 90):
        _, _, _, ctx = _ic_ctx(15, n_t, layout=hs.make_sensor_layout_3x3(grid))
        ctx.apply(v)
        tops.append(ctx.rank_trace[0])
    assert max(tops) <= 40 and max(tops) - min(tops) <= 5


def _source_ctx(n_side, n_t, layout=None):
    grid, op, K = _heat(n_side, n_t)
    cov = hs.CovarianceSpec.from_gamma(10.0, 1e4, grid)
    layout = layout if layout is not None else hs.full_observation(grid)
    return grid, op, K, hs.HessianContext(mode=hs.MODE_SOURCE, operator=K, layout=layout, cov=cov,
                                          pol=POL)


def test_source_hessian_zero_symmetry_and_dense_agreement():
    """test_hessian.py:172-208: zero -> rank 0; <Ha, b> = <a, Hb> to 1e-6; the stacked
    operator equals the dense brute force (1e-7 over 10 probes)."""
    grid, op, K, ctx = _source_ctx(5, 4)
    assert hs.misfit_apply_st(lp.LowRankMat.zeros(grid.n_x, 4), ctx).r == 0

    g15, _, K15, c15 = _source_ctx(15, 10, layout=hs.make_sensor_layout_3x3(lp.build_grid(15)))
    rng = np.random.default_rng(123)
    a, b = _field(rng, g15.n_x, 10, 2), _field(rng, g15.n_x, 10, 2)
    hab, ahb = lp.lr_dot(c15.apply(a), b), lp.lr_dot(a, c15.apply(b))
    assert abs(hab - ahb) <= 1e-6 * (abs(hab) + abs(ahb))

    Hd, _ = dense.dense_misfit_source(op.L.toarray(), grid.m_scale, K.time.tau, 4, ctx.layout.mask,
                                      ctx.cov.beta_noise, ctx.cov.gamma_prior)

    def stacked(v):
        X = np.asarray(v).reshape((grid.n_x, 4), order="F")
        return lp.lr_to_dense(ctx.apply(lp.lr_from_dense(X, POL))).reshape(-1, order="F")

    assert dense.hv_agreement(stacked, Hd, n_probe=10, seed=1) <= 1e-7


def test_steady_poisson_hessian_identities():
    """test_hessian.py:211-240: eigenpairs (beta_p/beta_n)/lambda^2 to 1e-10, zero maps to
    zero, the continuum limit 1e-4/(2 pi^2)^2 within 0.5% at n_side 127."""
    grid = lp.build_grid(15)
    op = lp.assemble_heat(grid)
    cov = hs.CovarianceSpec(1e4, 1.0, 1.0)
    for m, n in ((1, 1), (3, 2), (7, 5)):
        v = lp.eigvec_dense(m, n, grid)
        mu = 1e-4 / lp.discrete_fd_eig(m, n, grid) ** 2
        assert np.linalg.norm(hs.steady_poisson_apply(v, cov, op) - mu * v) <= 1e-10 * mu
    assert np.linalg.norm(hs.steady_poisson_apply(np.zeros(grid.n_x), cov, op)) == 0.0
    g127 = lp.build_grid(127)
    v = lp.eigvec_dense(1, 1, g127)
    mu_h = float(v @ hs.steady_poisson_apply(v, cov, lp.assemble_heat(g127)))
    target = 1e-4 / (2 * np.pi ** 2) ** 2
    assert abs(mu_h - target) / target < 5e-3


def test_hessians_are_self_adjoint_and_positive_semidefinite():
    """test_hessian.py:262-278 for the IC and the steady operator."""
    grid, op, K, ic = _ic_ctx(7, 4)
    rng = np.random.default_rng(124)
    for name, ctx in (("ic", ic), ("steady", _steady_ctx(7))):
        for _ in range(5):
            u, w = rng.standard_normal(grid.n_x), rng.standard_normal(grid.n_x)
            Hu, Hw = ctx.apply(u), ctx.apply(w)
            assert abs(float(Hu @ w) - float(u @ Hw)) <= 1e-6 * np.linalg.norm(Hu) * np.linalg.norm(w), name
            assert float(u @ Hu) >= -1e-10 * float(u @ u), name


# ================================================================ Arnoldi (test_arnoldi.py)
def test_identity_operator_breaks_down_in_the_first_step():
    """test_arnoldi.py:32-37."""
    v = np.ones(6) / np.sqrt(6)
    res = lp.lr_arnoldi(lambda x: x.copy() if isinstance(x, np.ndarray) else x.clone(), v, POL,
                        lp.StopRule(m_a=10))
    assert res.breakdown and res.iterations == 1
    assert res.H[0, 0] == pytest.approx(1.0, abs=1e-14)
    assert res.ritz_values[0].real == pytest.approx(1.0, abs=1e-12)


def test_zero_start_vector_is_rejected():
    """test_arnoldi.py:197-198."""
    with pytest.raises(ValueError):
        lp.lr_arnoldi(lambda x: x, np.zeros(4), POL, lp.StopRule(m_a=3))


def test_ritz_pairs_of_small_hessenbergs():
    """test_arnoldi.py:63-80: one column -> (h11, v1); a symmetric tridiagonal -> real pairs."""
    v = np.array([1.0, 0.0, 0.0])
    pairs = lp.ritz_pairs(np.array([[2.5], [0.0]]), [v])
    assert pairs[0][0] == pytest.approx(2.5)
    np.testing.assert_allclose(np.asarray(pairs[0][1]).ravel(), v)
    rng = np.random.default_rng(130)
    m = 12
    al, be = rng.standard_normal(m), np.abs(rng.standard_normal(m - 1)) + 0.1
    H = np.zeros((m + 1, m))
    H[:m, :m] = np.diag(al) + np.diag(be, 1) + np.diag(be, -1)
    pairs = lp.ritz_pairs(H, [c for c in np.eye(m).T])
    assert max(abs(complex(val).imag) for val, _ in pairs) == 0.0
    ref = np.sort(np.linalg.eigvalsh(H[:m, :m]))[::-1]
    np.testing.assert_allclose([complex(val).real for val, _ in pairs], ref, rtol=1e-10, atol=1e-12)


def test_ic_arnoldi_ritz_values_match_the_dense_top_40_after_restarts():
    """test_arnoldi.py:48-60, 162-175: full observation makes eigenvalues degenerate; with
    restart-on-breakdown the run recovers every multiplicity (1e-6 relative)."""
    grid, op, K, ctx = _ic_ctx(7, 5)
    Hd = _dense_ic(ctx, op, grid, K)
    ref = np.linalg.eigvalsh(Hd)[::-1]
    v1 = np.ones(grid.n_x) / np.sqrt(grid.n_x)
    res = lp.lr_arnoldi(ctx.apply, v1, POL,
                        lp.StopRule(m_a=57, eps_eig=1e-12, check_every=100, on_breakdown="restart"))
    assert res.restarts >= 1
    got = np.sort(res.ritz_values.real)[::-1][: len(ref)]
    assert np.max(np.abs(got[:40] - ref[:40]) / ref[:40]) <= 1e-6
    assert np.max(np.abs(got - ref) / ref) <= 1e-6


def test_ic_arnoldi_structure():
    """test_arnoldi.py:83-106: negligible imaginary parts, an orthonormal basis of unit
    vectors, and a Hessenberg matrix that is EXACTLY zero below the first subdiagonal."""
    grid, op, K, ctx = _ic_ctx(9, 6)
    v1 = np.ones(grid.n_x) / np.sqrt(grid.n_x)
    res = lp.lr_arnoldi(ctx.apply, v1, POL, lp.StopRule(m_a=25, eps_eig=1e-10, check_every=100))
    scale = np.abs(res.ritz_values.real).max()
    assert np.abs(res.ritz_values.imag).max() <= 1e-8 * scale
    assert res.gram_defect() <= 1e-6
    for b in res.basis:
        bn = b.cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
        assert abs(np.linalg.norm(bn) - 1.0) <= 1e-8
    H = res.H
    for j in range(H.shape[1]):
        assert (H[j + 2:, j] == 0.0).all()


def test_low_rank_arnoldi_relation():
    """test_arnoldi.py:125-141: H v_j = sum_i H[i,j] v_i within 10 eps0 ||H||, and one rank
    record per iteration (:109-122)."""
    grid, op, K, ctx = _source_ctx(7, 4)
    v1 = lp.LowRankMat(np.ones((grid.n_x, 1)), np.ones((4, 1)))
    res = lp.lr_arnoldi(ctx.apply, v1, POL, lp.StopRule(m_a=8, eps_eig=1e-14, check_every=100),
                        rank_source=ctx.rank_trace)
    assert len(res.rank_trace) == res.iterations
    Vd = [lp.lr_to_dense(b).ravel() for b in res.basis]
    hs_ = np.linalg.norm(res.H)
    for j in range(res.iterations):
        w = lp.lr_to_dense(ctx.apply(res.basis[j])).ravel()
        recon = sum(res.H[i, j] * Vd[i] for i in range(min(j + 2, len(Vd))))
        assert np.linalg.norm(w - recon) <= 10 * POL.eps0 * hs_


def test_top_ritz_value_grows_with_the_subspace_and_the_stop_rule_fires():
    """test_arnoldi.py:144-153, 178-185 on the steady operator (n_side 15)."""
    ctx = _steady_ctx(15)
    v1 = np.ones(ctx.n_param) / np.sqrt(ctx.n_param)
    tops = []
    for m_a in (4, 8, 16, 32):
        res = lp.lr_arnoldi(ctx.clone().apply, v1, POL,
                            lp.StopRule(m_a=m_a, eps_eig=1e-14, check_every=100))
        tops.append(res.ritz_values.real[0])
    slack = 10 * POL.eps0 * tops[-1]
    assert all(b >= a - slack for a, b in zip(tops, tops[1:]))
    res = lp.lr_arnoldi(ctx.apply, v1, POL, lp.StopRule(m_a=200, eps_eig=1e-9, check_every=5))
    assert res.iterations < 200 and res.converged_count >= 1


def test_degenerate_pair_spans_the_right_subspace():
    """test_arnoldi.py:156-169: modes (1,2)/(2,1) share an eigenvalue; the two Ritz vectors
    span their plane to 1e-5 rad."""
    ctx = _steady_ctx(15)
    grid = lp.build_grid(15)
    v1 = np.ones(ctx.n_param) / np.sqrt(ctx.n_param)
    res = lp.lr_arnoldi(ctx.apply, v1, POL,
                        lp.StopRule(m_a=80, eps_eig=1e-14, check_every=100, on_breakdown="restart"))
    vals = res.ritz_values.real
    assert vals[1] == pytest.approx(vals[2], rel=1e-10)
    as_np = lambda x: x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)  # noqa: E731
    Vr = np.column_stack([as_np(res.ritz_vectors[1]).ravel(), as_np(res.ritz_vectors[2]).ravel()])
    Va = np.column_stack([lp.eigvec_dense(1, 2, grid), lp.eigvec_dense(2, 1, grid)])
    assert sla.subspace_angles(Vr, Va).max() <= 1e-5


def test_rank_one_check_on_separable_and_mixed_modes():
    """test_arnoldi.py:201-227."""
    grid = lp.build_grid(15)
    r, ratio = lp.rank_one_check(lp.eigvec_dense(2, 3, grid), reshape=(15, 15))
    assert r == 1 and ratio <= 1e-6
    two = lp.eigvec_dense(1, 1, grid) + lp.eigvec_dense(2, 2, grid)
    r, ratio = lp.rank_one_check(two, reshape=(15, 15))
    assert r == 2 and ratio > 0.1
    r, _ = lp.rank_one_check(np.random.default_rng(131).standard_normal(225), reshape=(15, 15))
    assert r >= 13
    rng = np.random.default_rng(132)
    A = lp.LowRankMat(rng.standard_normal((20, 2)), rng.standard_normal((9, 2)))
    r, ratio = lp.rank_one_check(A)
    assert r == 2 and ratio > 0


# ================================================================ posterior (test_posterior.py)
def _orthonormal(rng, n, k):
    return np.linalg.qr(rng.standard_normal((n, k)))[0]


def test_no_retained_pair_gives_the_prior_and_a_huge_one_localises():
    """test_posterior.py:29-42."""
    s = posterior.build_summary(np.array([]), [], gamma_prior=10.0, eps_eig=0.1, n_x=25)
    assert s.k == 0
    np.testing.assert_allclose(s.variance_field, 10.0)
    var = posterior.variance_diag(np.array([1e12]), np.eye(16)[:, [0]], gamma_prior=10.0)
    assert var[0] <= 1e-9
    np.testing.assert_allclose(var[1:], 10.0)


def test_variance_and_posterior_action_match_the_dense_inverse():
    """test_posterior.py:45-59, 79-99 (1e-4): full eigendecomposition of the dense H."""
    grid, op, K, ctx = _ic_ctx(7, 5)
    Hd = _dense_ic(ctx, op, grid, K)
    w, V = np.linalg.eigh(Hd)
    s = posterior.build_summary(w[::-1].astype(complex), list(V[:, ::-1].T), gamma_prior=10.0,
                                eps_eig=1e-8)
    ref_diag = np.asarray(dense.dense_posterior_diag(Hd, 10.0))
    assert np.max(np.abs(s.variance_field - ref_diag) / ref_diag) <= 1e-4
    post = sla.inv(Hd / 10.0 + np.eye(grid.n_x) / 10.0)
    rng = np.random.default_rng(140)
    for _ in range(5):
        v = rng.standard_normal(grid.n_x)
        assert np.linalg.norm(posterior.posterior_apply(v, s) - post @ v) <= 1e-4 * np.linalg.norm(post @ v)


def test_posterior_action_special_cases():
    """test_posterior.py:62-76: empty summary = gamma I; an eigenvector is scaled by
    gamma (1 - lambda/(1+lambda))."""
    rng = np.random.default_rng(141)
    n = 30
    empty = posterior.build_summary(np.array([]), [], gamma_prior=7.0, eps_eig=0.1, n_x=n)
    v = rng.standard_normal(n)
    np.testing.assert_allclose(posterior.posterior_apply(v, empty), 7.0 * v)
    V = _orthonormal(rng, n, 3)
    s = posterior.build_summary(np.array([4.0, 2.0, 1.0], dtype=complex), list(V.T), gamma_prior=7.0)
    np.testing.assert_allclose(posterior.posterior_apply(V[:, 0], s), 7.0 * (1 - 0.8) * V[:, 0],
                               atol=1e-12)


def test_variance_monotonicity_properties():
    """test_posterior.py:102-126: 0 < var <= gamma; another retained pair never raises it;
    larger eigenvalues (more noise weight) lower it wherever the vectors have support."""
    rng = np.random.default_rng(142)
    V = _orthonormal(rng, 40, 6)
    lams = np.sort(rng.uniform(0.05, 40.0, 6))[::-1]
    var = posterior.variance_diag(lams, V, gamma_prior=10.0)
    assert (var <= 10.0 + 1e-12).all() and (var > 0).all()
    fewer = posterior.variance_diag(lams[:3], V[:, :3], gamma_prior=10.0)
    more = posterior.variance_diag(lams[:5], V[:, :5], gamma_prior=10.0)
    assert (more <= fewer + 1e-12).all()
    scaled = posterior.variance_diag(100.0 * lams, V, gamma_prior=10.0)
    hit = (V ** 2).sum(axis=1) > 1e-12
    assert (scaled[hit] < var[hit]).all()


def test_retention_threshold_and_reorthonormalisation():
    """test_posterior.py:129-149: pairs below eps_eig are dropped, filters descend; a nearly
    duplicated direction does not double-count (variance stays positive)."""
    rng = np.random.default_rng(143)
    V = _orthonormal(rng, 20, 4)
    s = posterior.build_summary(np.array([5.0, 0.5, 0.05, 0.005], dtype=complex), list(V.T),
                                gamma_prior=1.0, eps_eig=0.1)
    assert s.k == 2
    np.testing.assert_allclose(s.eigenvalues, [5.0, 0.5])
    assert (np.diff(s.filters) <= 0).all()
    v = _orthonormal(rng, 25, 1)[:, 0]
    dup = np.column_stack([v, v + 1e-7 * rng.standard_normal(25)])
    assert posterior.variance_diag(np.array([10.0, 10.0]), dup, gamma_prior=1.0).min() > 0


def test_variance_drops_at_every_sensor_node():
    """test_posterior.py:152-162 through the device Arnoldi: heat 31^2, n_t 10, 3x3 sensors,
    m_a 25, eps_eig 0.1 — strictly below the prior at the sensors, never above it."""
    grid = lp.build_grid(31)
    layout = hs.make_sensor_layout_3x3(grid)
    _, _, _, ctx = _ic_ctx(31, 10, layout=layout)
    v1 = np.ones(grid.n_x) / np.sqrt(grid.n_x)
    res = lp.lr_arnoldi(ctx.apply, v1, POL, lp.StopRule(m_a=25, eps_eig=1e-1, check_every=10))
    s = posterior.build_summary(res.ritz_values, res.ritz_vectors, gamma_prior=10.0, eps_eig=1e-1)
    assert s.k >= 1
    assert (s.variance_field[layout.mask] < 10.0).all()
    assert (s.variance_field <= 10.0 + 1e-12).all()


# ================================================================ dense cross-check (test_oracle.py)
def test_dense_hessian_basic_facts():
    """test_oracle.py:24-63: no sensors -> the zero matrix; symmetric to 1e-10; its trace is
    the sum of e_i . H e_i through the device path; positive semidefinite."""
    grid, op, K, ctx = _ic_ctx(5, 3)
    Hz, dz = dense.dense_misfit_ic(op.L.toarray(), grid.m_scale, K.time.tau, 3,
                                   np.zeros(grid.n_x, dtype=bool), ctx.cov.beta_noise,
                                   ctx.cov.gamma_prior)
    assert np.abs(Hz).max() == 0.0 and dz == 0.0
    grid, op, K, ctx = _ic_ctx(7, 5)
    Hd, defect = dense.dense_misfit_ic(op.L.toarray(), grid.m_scale, K.time.tau, 5, ctx.layout.mask,
                                       ctx.cov.beta_noise, ctx.cov.gamma_prior)
    assert defect <= 1e-10
    E = np.eye(grid.n_x)
    diag_sum = sum(float(E[i] @ ctx.apply(E[i])) for i in range(grid.n_x))
    assert abs(np.trace(Hd) - diag_sum) <= 1e-10 * abs(diag_sum)
    w = np.linalg.eigvalsh(Hd)
    assert w.min() >= -1e-12 * w.max()
    post = dense.dense_posterior_diag(Hd, ctx.cov.gamma_prior)
    assert (post <= ctx.cov.gamma_prior + 1e-12).all() and (post > 0).all()   # :116-121


def test_dense_hessian_equals_the_kronecker_system():
    """test_oracle.py:66-83 restated for the Hessian: H = g m^2 w E0^T K^-T (I (x) diag(mask))
    K^-1 E0 with the full space-time matrix assembled and solved directly."""
    grid, op, K = _heat(5, 3)
    n, n_t, tau, m = grid.n_x, 3, K.time.tau, grid.m_scale
    A = m * (np.eye(n) + tau * op.L.toarray())
    Kfull = np.kron(np.eye(n_t), A) - m * np.kron(np.diag(np.ones(n_t - 1), -1), np.eye(n))
    mask = np.random.default_rng(150).random(n) < 0.4
    bn, g = 3e3, 2.0
    E0 = np.zeros((n * n_t, n))
    E0[:n] = np.eye(n)
    Y = np.linalg.solve(Kfull, m * np.sqrt(g) * E0)
    W = np.kron(np.eye(n_t), np.diag(mask.astype(float))) * (bn * tau * m)
    ref = np.sqrt(g) * m * (np.linalg.solve(Kfull.T, W @ Y))[:n]
    Hd, _ = dense.dense_misfit_ic(op.L.toarray(), m, tau, n_t, mask, bn, g)
    assert np.abs(Hd - 0.5 * (ref + ref.T)).max() <= 1e-10 * np.abs(ref).max()


def test_dense_eigensolver_and_size_cap():
    """test_oracle.py:86-107, 124-131."""
    vals, vecs = dense.dense_eig_top(np.diag([3.0, 2.0, 1.0]), 2)
    np.testing.assert_allclose(vals, [3.0, 2.0])
    np.testing.assert_allclose(np.abs(vecs), np.eye(3)[:, :2], atol=1e-14)
    grid = lp.build_grid(3)
    vals, _ = dense.dense_eig_top(lp.assemble_heat(grid).L.toarray(), 9)
    formula = np.sort([lp.discrete_fd_eig(m, n, grid) for m in range(1, 4) for n in range(1, 4)])[::-1]
    np.testing.assert_allclose(vals, formula, rtol=1e-12)
    with pytest.raises(lp.InvalidConfigError):
        dense.dense_eig_top(np.array([[0.0, 1.0], [0.0, 0.0]]), 1)
    with pytest.raises(lp.InvalidConfigError):
        dense.dense_misfit_ic(np.eye(2500), 1.0, 0.1, 3, np.ones(2500, dtype=bool), 1.0, 1.0)
    with pytest.raises(lp.InvalidConfigError):
        dense.dense_misfit_source(np.eye(900), 1.0, 0.1, 3, np.ones(900, dtype=bool), 1.0, 1.0)


def test_steady_dense_matrix_has_the_formula_eigenpair():
    """test_oracle.py:174-182."""
    grid = lp.build_grid(5)
    Hd, defect = dense.dense_misfit_steady(lp.assemble_heat(grid).L.toarray(), 1e4, 1.0)
    assert defect <= 1e-12
    v = lp.eigvec_dense(1, 1, grid)
    mu = 1e-4 / lp.discrete_fd_eig(1, 1, grid) ** 2
    assert np.linalg.norm(Hd @ v - mu * v) <= 1e-10 * mu


def test_compare_reports():
    """test_oracle.py:134-171: self-comparison is exact; a 1e-3 eigenvalue error fails the
    gate; a rotated degenerate pair passes (cluster-wise principal angles)."""
    rng = np.random.default_rng(151)
    A = rng.standard_normal((12, 12))
    Hd = A @ A.T
    vals, vecs = dense.dense_eig_top(Hd, 5)
    diag = dense.dense_posterior_diag(Hd, 1.0)
    rep = dense.compare(vals, vecs, vals, vecs, Hd=Hd, lr_variance=diag, dense_variance=diag,
                        hv_rel_error=0.0)
    assert rep.passed and rep.max_eig_rel_error == 0.0 and rep.variance_rel_error == 0.0
    assert rep.max_principal_angle <= 1e-7
    bad = dense.compare(vals * (1 + 1e-3), vecs, vals, vecs)
    assert not bad.passed and bad.max_eig_rel_error >= 0.99e-3
    v4 = np.array([2.0, 1.0, 1.0, 0.5])
    V = np.linalg.qr(rng.standard_normal((8, 4)))[0]
    c, s = np.cos(0.7), np.sin(0.7)
    R = np.eye(4)
    R[1:3, 1:3] = [[c, -s], [s, c]]
    assert dense.compare(v4, V @ R, v4, V).max_principal_angle <= 1e-10


def test_dense_substitution_solves_the_kronecker_system_both_ways():
    """test_oracle.py:66-83: dense_forward against the assembled space-time matrix, forward
    and adjoint (1e-10)."""
    grid, op, _ = _heat(5, 3)
    n, n_t, tau, m = grid.n_x, 3, 1.0 / 3.0, grid.m_scale
    A = m * (np.eye(n) + tau * op.L.toarray())
    Kfull = np.kron(np.eye(n_t), A) - m * np.kron(np.diag(np.ones(n_t - 1), -1), np.eye(n))
    F = np.random.default_rng(152).standard_normal((n, n_t))
    Y = dense.dense_forward(op.L.toarray(), m, tau, F)
    np.testing.assert_allclose(Y.reshape(-1, order="F"),
                               np.linalg.solve(Kfull, F.reshape(-1, order="F")), rtol=1e-10)
    Z = dense.dense_forward(op.L.toarray(), m, tau, F, adjoint=True)
    np.testing.assert_allclose(Z.reshape(-1, order="F"),
                               np.linalg.solve(Kfull.T, F.reshape(-1, order="F")), rtol=1e-10)
    # and the device sweep solves the same system
    K = lp.SpaceTimeOperator(op, lp.build_time_grid(n_t))
    S = lp.lr_to_dense(lp.st_solve_sweep(K, lp.lr_from_dense(F, POL), POL))
    assert np.linalg.norm(S - Y) <= 1e-8 * np.linalg.norm(Y)
