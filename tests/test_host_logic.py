"""Host-side logic of the package (no GPU): the validation, layouts, scalar
identities and discretisation facts the reference's unit tests pin, through
the same public names.  Each test cites the reference test whose behaviour it
mirrors; everything that computes on fields lives in the -m gpu files."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_1703_05638_b200 as lp
from paper_1703_05638_b200 import hessian as hs
from paper_1703_05638_b200 import posterior

POL = lp.TruncationPolicy(1e-8)


# ------------------------------------------------------------------ policies, factors
def test_truncation_policy_bounds():
    """test_lowrank.py:25-31: eps0 in (0,1), r_max >= 0 (0 is a legal cap)."""
    for bad in (0.0, 1.0, -1e-3, 2.0):
        with pytest.raises(ValueError):
            lp.TruncationPolicy(bad)
    with pytest.raises(ValueError):
        lp.TruncationPolicy(1e-8, -1)
    assert lp.TruncationPolicy(1e-8, 0).r_max == 0
    assert lp.TruncationPolicy().eps0 == 1e-8 and lp.TruncationPolicy().r_max is None


def test_factor_shape_mismatch_is_a_value_error_without_a_device():
    """test_lowrank.py:34-36; the check runs before any device call."""
    with pytest.raises(ValueError):
        lp.LowRankMat(np.zeros((6, 2)), np.zeros((5, 3)))
    with pytest.raises(ValueError):
        lp.LowRankMat(np.zeros((6, 2, 1)), np.zeros((5, 2)))


def test_stop_rule_rejects_bad_settings():
    """test_arnoldi.py:190-196."""
    for kw in (dict(m_a=0), dict(m_a=4, eps_eig=0.0), dict(m_a=4, eps_eig=-1.0),
               dict(m_a=4, on_breakdown="explode")):
        with pytest.raises(ValueError):
            lp.StopRule(**kw)
    s = lp.StopRule(m_a=7)
    assert (s.eps_eig, s.check_every, s.on_breakdown) == (1e-1, 10, "stop")


def test_rank_one_check_needs_a_reshape_for_dense_input():
    """test_arnoldi.py:229-231."""
    with pytest.raises(ValueError):
        lp.rank_one_check(np.ones(9))


# ------------------------------------------------------------------ covariance, sensors
def test_covariance_presets_share_one_identity():
    """test_hessian.py:24-30: gamma * beta_prior * h^d = 1 from either preset."""
    grid = lp.build_grid(23)
    a = hs.CovarianceSpec.from_gamma(4.0, 2.5e3, grid)
    b = hs.CovarianceSpec.from_beta(a.beta_prior, 2.5e3, grid)
    assert a.gamma_prior * a.beta_prior * grid.m_scale == pytest.approx(1.0, rel=1e-14)
    assert b.gamma_prior == pytest.approx(a.gamma_prior, rel=1e-14)
    assert a.beta_noise == pytest.approx(2.5e3 * a.beta_prior, rel=1e-14)
    assert b.beta_noise == pytest.approx(a.beta_noise, rel=1e-14)


def test_covariance_rejects_nonpositive_scalars():
    """test_hessian.py:32-37."""
    for bn, bp, g in ((0.0, 1.0, 1.0), (1.0, -2.0, 1.0), (1.0, 1.0, 0.0)):
        with pytest.raises(lp.InvalidConfigError):
            hs.CovarianceSpec(bn, bp, g)


@pytest.mark.parametrize("n_side,count", [(63, 144), (31, 36), (15, 9)])
def test_3x3_layout_counts(n_side, count):
    """test_hessian.py:41-47: nine square dof blocks (4x4 at 63, 2x2 at 31, 1x1 at 15)."""
    assert hs.make_sensor_layout_3x3(lp.build_grid(n_side)).n_active == count


def test_3x3_patches_do_not_overlap():
    """test_hessian.py:49-55."""
    for n_side in (15, 31, 63, 127):
        grid = lp.build_grid(n_side)
        whole = hs.make_sensor_layout_3x3(grid)
        parts = [hs.make_sensor_layout([p], grid).mask for p in whole.patches]
        assert sum(int(m.sum()) for m in parts) == whole.n_active
        assert np.array_equal(np.logical_or.reduce(parts), whole.mask)


def test_layout_errors():
    """test_hessian.py:57-66: too coarse a grid, a patch outside the domain."""
    with pytest.raises(lp.InvalidConfigError):
        hs.make_sensor_layout_3x3(lp.build_grid(7))
    with pytest.raises(lp.InvalidConfigError):
        hs.make_sensor_layout([(0.5, 0.5, 1e-3)], lp.build_grid(4))
    with pytest.raises(lp.InvalidConfigError):
        hs.make_sensor_layout([(1.2, 0.5, 0.1)], lp.build_grid(15))


def test_full_empty_and_subgrid_layouts():
    grid = lp.build_grid(16)
    assert hs.full_observation(grid).n_active == grid.n_x
    assert hs.empty_observation(grid).n_active == 0
    sub = hs.make_sensor_subgrid(grid, 4)
    assert sub.n_active == 16
    # 0-based indices stride/2 + stride*j per axis
    idx = np.flatnonzero(sub.mask)
    assert set(idx % 16) == {2, 6, 10, 14} and set(idx // 16) == {2, 6, 10, 14}
    g3 = lp.build_grid(8, 3)
    assert hs.make_sensor_subgrid(g3, 4).n_active == 64


def test_steady_mode_is_defined_for_the_heat_operator_only():
    """test_hessian.py:243-249."""
    cd = lp.assemble_convdiff(lp.build_grid(5), 1e-2, (0.0, 1.0))
    with pytest.raises(lp.InvalidConfigError):
        hs.HessianContext(mode=hs.MODE_STEADY, operator=None, layout=None,
                          cov=hs.CovarianceSpec(1e4, 1.0, 1.0), pol=POL, spatial=cd)


# ------------------------------------------------------------------ posterior scalars
def test_filter_factor_values_and_sign_check():
    """test_posterior.py:13-21: lambda / (1 + lambda); negative input is a NumericalError."""
    assert posterior.lambda_tilde(0.0) == 0.0
    assert posterior.lambda_tilde(1.0) == 0.5
    assert posterior.lambda_tilde(3.0) == 0.75
    assert posterior.lambda_tilde(1e6) == pytest.approx(1e6 / (1e6 + 1.0), rel=1e-15)
    with pytest.raises(lp.NumericalError):
        posterior.lambda_tilde(-1e-3)


def test_summary_refuses_a_complex_spectrum():
    """test_posterior.py:137-140 (checked on the host before any device work)."""
    with pytest.raises(lp.NumericalError):
        posterior.build_summary(np.array([1.0 + 0.1j, 0.5]), [np.ones(4), np.ones(4)],
                                gamma_prior=1.0)


# ------------------------------------------------------------------ discretisation
def test_grid_and_time_grid_scalars():
    """discretize.py:3-6, 75-87: h = 1/(n+1), M = h^d, tau = T/n_t."""
    g = lp.build_grid(9)
    assert (g.n_x, g.h, g.m_scale) == (81, 0.1, pytest.approx(0.01))
    g3 = lp.build_grid(4, 3)
    assert g3.n_x == 64 and g3.m_scale == pytest.approx(0.2 ** 3)
    tg = lp.build_time_grid(8, T=2.0)
    assert (tg.n_t, tg.tau, tg.T) == (8, 0.25, 2.0)
    for bad in (0, -3):
        with pytest.raises((ValueError, lp.InvalidConfigError)):
            lp.build_grid(bad)
        with pytest.raises((ValueError, lp.InvalidConfigError)):
            lp.build_time_grid(bad)


def test_heat_matrix_is_the_five_point_laplacian():
    """test_discretize.py:93-109: symmetric, <= 5 entries per row, 4/h^2 on the diagonal,
    eigenpairs given by the FD formula."""
    grid = lp.build_grid(6)
    L = sp.csr_matrix(lp.assemble_heat(grid).L)
    assert abs(L - L.T).max() == 0.0
    assert np.diff(L.indptr).max() <= 5
    np.testing.assert_allclose(L.diagonal(), 4.0 / grid.h ** 2, rtol=1e-15)
    for m, n in ((1, 1), (2, 5), (6, 6)):
        v = lp.eigvec_dense(m, n, grid)
        assert np.linalg.norm(v) == pytest.approx(1.0, rel=1e-13)
        lam = lp.discrete_fd_eig(m, n, grid)
        assert np.linalg.norm(L @ v - lam * v) <= 1e-11 * lam
    # h -> 0: the discrete eigenvalue approaches pi^2 (m^2 + n^2) from below
    fine = lp.discrete_fd_eig(1, 1, lp.build_grid(255))
    assert 0 < lp.analytic_poisson_eig(1, 1) - fine < 1e-3 * fine
    with pytest.raises((ValueError, lp.InvalidConfigError)):
        lp.discrete_fd_eig(0, 1, grid)
    with pytest.raises((ValueError, lp.InvalidConfigError)):
        lp.discrete_fd_eig(1, 7, grid)


def test_q1_and_3d_heat_matrices_match_their_closed_form_eigenvalues():
    """lumped-mass Q1 and the 3-D 7-point operator on separable sine modes."""
    g = lp.build_grid(7)
    Lq = sp.csr_matrix(lp.assemble_heat(g, "q1").L)
    assert abs(Lq - Lq.T).max() < 1e-12 * abs(Lq).max() and np.diff(Lq.indptr).max() <= 9
    v = lp.eigvec_dense(2, 3, g)
    lam = lp.discretize.operator_eig(g, (2, 3), "q1")
    assert np.linalg.norm(Lq @ v - lam * v) <= 1e-11 * lam
    g3 = lp.build_grid(5, 3)
    L3 = sp.csr_matrix(lp.assemble_heat(g3).L)
    assert np.diff(L3.indptr).max() <= 7
    x = np.sin(np.pi * np.arange(1, 6) / 6)
    v3 = np.einsum("k,j,i->kji", np.sin(2 * np.pi * np.arange(1, 6) / 6), x, x).ravel()
    lam3 = lp.discretize.operator_eig(g3, (1, 1, 2), "fd")
    assert np.linalg.norm(L3 @ v3 - lam3 * v3) <= 1e-11 * lam3 * np.linalg.norm(v3)


def test_upwind_convdiff_rows_follow_the_wind_sign():
    """test_discretize.py (upwind): nu * Laplacian + first-order upwind, so the matrix is an
    M-matrix (positive diagonal, nonpositive off-diagonals) and reduces to heat at w = 0."""
    grid = lp.build_grid(8)
    for w in ((0.7, -1.3), (-0.4, 0.0), (0.0, 2.0)):
        A = sp.csr_matrix(lp.assemble_convdiff(grid, 0.05, w).L)
        off = A - sp.diags(A.diagonal())
        assert A.diagonal().min() > 0 and off.max() <= 0.0
        # upstream neighbour carries the convective weight: for w_x > 0 the west entry is larger
        i = 3 * 8 + 4
        west, east = -A[i, i - 1], -A[i, i + 1]
        assert (west > east) == (w[0] > 0) or w[0] == 0.0
    H = sp.csr_matrix(lp.assemble_heat(grid).L)
    Z = sp.csr_matrix(lp.assemble_convdiff(grid, 1.0, (0.0, 0.0)).L)
    assert abs(H - Z).max() <= 1e-12 * abs(H).max()


def test_galerkin_convection_is_skew_for_a_constant_wind():
    """D3: N_ij = int (w . grad phi_j) phi_i is exactly skew-symmetric for a constant
    wind and zero Dirichlet data, so S's symmetric part is the diffusion operator's."""
    grid = lp.build_grid(9)
    nu = 0.05
    A = sp.csr_matrix(lp.assemble_convdiff(grid, nu, (0.6, -0.9), scheme="galerkin").L)
    D = sp.csr_matrix(lp.assemble_convdiff(grid, nu, (0.0, 0.0), scheme="galerkin").L)
    N = A - D
    assert abs(N + N.T).max() <= 1e-12 * abs(N).max()
    assert abs(N).max() > 0 and np.diff(A.indptr).max() <= 9


def test_oracle_report_text_round_trip():
    """test_oracle.py:160-171: key=value lines, result=PASS, values parse back."""
    from paper_1703_05638_b200 import dense

    rep = dense.OracleReport(eig_rel_errors=np.array([1e-9]), max_eig_rel_error=1e-9,
                             max_principal_angle=2e-7, max_pair_residual=3e-9,
                             variance_rel_error=4e-6, hv_rel_error=5e-10,
                             tolerances={"eig_rel": 1e-6}, passed=True)
    text = rep.as_text()
    assert "result=PASS" in text
    parsed = dict(line.split("=") for line in text.strip().splitlines())
    assert float(parsed["max_eig_rel_error"]) == pytest.approx(1e-9)
    assert float(parsed["variance_rel_error"]) == pytest.approx(4e-6)
    assert float(parsed["tol_eig_rel"]) == pytest.approx(1e-6)


def test_dof_indexing_and_coordinates():
    """test_discretize.py:21-33: (i, j) <-> dof is a bijection with x1 fastest; coords follow it."""
    g = lp.build_grid(6)
    seen = {g.ij_to_dof(i, j) for i in range(6) for j in range(6)}
    assert seen == set(range(36))
    for k in (0, 5, 6, 17, 35):
        assert g.ij_to_dof(*g.dof_to_ij(k)) == k
    x1, x2 = g.coords()
    k = g.ij_to_dof(4, 2)
    assert x1[k] == pytest.approx(5 * g.h) and x2[k] == pytest.approx(3 * g.h)


def test_laplacian_of_ones_vanishes_away_from_the_boundary():
    """test_discretize.py:53-62."""
    g = lp.build_grid(9)
    out = (sp.csr_matrix(lp.assemble_heat(g).L) @ np.ones(g.n_x)).reshape(9, 9)
    assert np.abs(out[1:-1, 1:-1]).max() <= 1e-10 * (4 / g.h ** 2)
    assert (out[0] > 0).all() and (out[:, -1] > 0).all()


def test_convdiff_validation_and_row_sums():
    """test_discretize.py:73-96: nu > 0 required; upwinding keeps row sums nonnegative and the
    symmetric part positive definite; at most five entries per row."""
    g = lp.build_grid(7)
    for nu in (0.0, -1e-2):
        with pytest.raises(lp.InvalidConfigError):
            lp.assemble_convdiff(g, nu, (0.0, 1.0))
    for w in ((1.0, 0.0), (-0.5, 2.0), (0.3, -0.7)):
        A = sp.csr_matrix(lp.assemble_convdiff(g, 1e-2, w).L)
        assert np.asarray(A.sum(axis=1)).min() >= -1e-9 * abs(A).max()
        assert np.linalg.eigvalsh(0.5 * (A + A.T).toarray())[0] > 0
        assert np.diff(A.indptr).max() <= 5


def test_discrete_eigenvalues_order_and_mode_symmetries():
    """test_discretize.py:98-141: pi^2 (m^2/a^2 + n^2/b^2); the discrete values increase with
    either index; the first mode is positive; even modes are antisymmetric under reflection."""
    assert lp.analytic_poisson_eig(1, 1) == pytest.approx(2 * np.pi ** 2, rel=1e-15)
    assert lp.analytic_poisson_eig(2, 3, a=2.0, b=0.5) == pytest.approx(np.pi ** 2 * (1.0 + 36.0))
    g = lp.build_grid(9)
    vals = np.array([[lp.discrete_fd_eig(m, n, g) for n in range(1, 10)] for m in range(1, 10)])
    assert (np.diff(vals, axis=0) > 0).all() and (np.diff(vals, axis=1) > 0).all()
    assert (lp.eigvec_dense(1, 1, g) > 0).all()
    v = lp.eigvec_dense(2, 1, g).reshape(9, 9)       # row j = x2 level, column i = x1
    np.testing.assert_allclose(v, -v[:, ::-1], atol=1e-14)
    f1, f2 = lp.analytic_separable_eigvec(2, 3, g)
    np.testing.assert_allclose(np.outer(f2, f1).ravel() / np.linalg.norm(np.outer(f2, f1)),
                               lp.eigvec_dense(2, 3, g), atol=1e-14)


def test_coo_text_exchange_round_trip(tmp_path):
    """test_discretize.py:153-158: bit-exact through the 17-digit text form."""
    from paper_1703_05638_b200 import discretize as dz

    op = lp.assemble_convdiff(lp.build_grid(5), 3e-2, (0.2, 1.0))
    dz.export_coo(op, tmp_path / "op.coo")
    back = dz.import_coo(tmp_path / "op.coo", op.grid.n_x)
    assert np.abs((back - op.L).toarray()).max() == 0.0


def test_variance_writers(tmp_path):
    """test_posterior.py:165-195: CSV grid with header, 17 digits; PGM maps the minimum to 0 and
    gamma to 255; a flat field at the prior is all white."""
    rng = np.random.default_rng(7)
    n = 6
    field = rng.uniform(2.0, 10.0, n * n)
    field[13] = 1.0
    posterior.write_variance_csv(field, n, tmp_path / "v.csv")
    posterior.write_variance_pgm(field, n, 10.0, tmp_path / "v.pgm")
    rows = (tmp_path / "v.csv").read_text().strip().splitlines()
    assert len(rows) == n + 1 and rows[0] == ",".join(f"c{i}" for i in range(n))
    back = np.array([[float(x) for x in r.split(",")] for r in rows[1:]])
    np.testing.assert_array_equal(back.ravel(), field)
    np.testing.assert_array_equal(posterior.variance_to_grid(field, n), back)
    pgm = (tmp_path / "v.pgm").read_text().split()
    assert pgm[:4] == ["P2", str(n), str(n), "255"]
    pix = np.array(pgm[4:], dtype=int)
    assert pix.size == n * n and pix.min() == 0 and pix[13] == 0 and pix.max() <= 255
    posterior.write_variance_pgm(np.full(9, 10.0), 3, 10.0, tmp_path / "flat.pgm")
    assert all(p == "255" for p in (tmp_path / "flat.pgm").read_text().split()[4:])
