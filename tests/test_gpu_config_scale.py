"""GPU parity at the BASELINE configuration sizes, against fixtures the
REFERENCE produced (tests/golden/make_golden_config.py, config_*.npz).

North-star tolerances (BASELINE.json): leading Hessian eigenvalues to relative
1e-6, pointwise posterior variance to relative 1e-5, Krylov iteration counts
within ±1.  Single applies: relative 1e-9 on H̃v (the reference agrees with the
dense brute force to 1e-8, test_hessian.py:117-127; the device path computes
the same truncations in an orthogonally equivalent basis) and IDENTICAL rank
traces (every flush of both sweeps and the observation truncation).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_05638_b200 as lp  # noqa: E402
from oracle import lrk_oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _fx(name):
    return dict(np.load(os.path.join(HERE, "golden", f"config_{name}.npz")))


def _ctx(n_side, dim, stencil, n_t, per_axis, every, sigma, delta, gp, rmax, mode="ic",
         full=False):
    grid = lp.build_grid(n_side, dim)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid, stencil), lp.build_time_grid(n_t))
    bn = 1.0 / (sigma ** 2 * K.time.tau * grid.m_scale)  # w = 1/σ²
    cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=delta, prior_gamma=gp)
    layout = (lp.SensorLayout((), np.ones(grid.n_x, bool), time_every=every) if full
              else lp.make_sensor_subgrid(grid, per_axis, time_every=every))
    return lp.HessianContext(mode=mode, operator=K, layout=layout, cov=cov,
                             pol=lp.TruncationPolicy(1e-8, rmax)), grid, bn


def _c2():
    return _ctx(256, 2, "q1", 512, 32, 1, 0.01, 1.0, 0.05, 32)


def _check_apply(ctx, v, fx):
    out = ctx.apply(v)
    ref = fx["O"]
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    fw, ob, bw = ctx.last_traces()
    assert fw == fx["fwd"].tolist(), "forward-sweep rank trace differs from the reference"
    assert bw == fx["bwd"].tolist(), "adjoint-sweep rank trace differs from the reference"
    assert ob == int(fx["obs"][0])
    assert ctx.rank_trace[-1] == int(fx["max_rank"][0])
    assert err <= 1e-9, err


@pytest.mark.parametrize("form", ["auto", "persistent", "streaming"])
def test_c2_apply_at_bench_config_vs_reference(monkeypatch, form):
    """The EXACT C2 workload (Q1 256², n_t 512, 32×32 sensors, prior, r_max
    32): one apply against the reference, identical per-flush ranks — with
    either sweep form (persistent resident-row kernel / streaming flush)."""
    if form != "auto":
        monkeypatch.setenv("LRK_SFLUSH", "0" if form == "persistent" else "1")
    ctx, grid, _ = _c2()
    fx = _fx("c2_apply")
    v = np.random.default_rng(1).standard_normal(grid.n_x)
    _check_apply(ctx, v / np.linalg.norm(v), fx)


def test_c2_arnoldi_eigenvalues_and_variance_vs_reference():
    """C2 eigen run with the reference's default stop rule (m_a 50, eps_eig 0.1,
    check_every 10): iterations ±1, retained eigenvalues to 1e-6, posterior
    variance with the config prior to 1e-5 (and its reduction γ − var)."""
    ctx, grid, _ = _c2()
    fx = _fx("c2_arnoldi")
    v1 = np.random.default_rng(1).standard_normal(grid.n_x)
    v1 /= np.linalg.norm(v1)
    res = lp.lr_arnoldi(ctx.apply, v1, ctx.pol, lp.StopRule(m_a=50, eps_eig=1e-1, check_every=10),
                        rank_source=ctx.rank_trace)
    assert abs(res.iterations - int(fx["iters"][0])) <= 1
    ref = fx["retained"]
    got = np.sort(res.ritz_values.real[res.ritz_values.real >= 1e-1])[::-1]
    n = min(len(ref), len(got))
    assert abs(len(ref) - len(got)) <= 1
    np.testing.assert_allclose(got[:n], ref[:n], rtol=1e-6)
    summ = lp.build_summary(res.ritz_values, res.ritz_vectors, 1.0, 1e-1, prior=ctx.prior)
    np.testing.assert_allclose(summ.variance_field, fx["var"], rtol=1e-5)
    diag = ctx.prior.diag(2).cpu().numpy()
    red = diag - summ.variance_field
    assert np.abs(red - fx["reduction"]).max() <= 1e-5 * np.abs(fx["reduction"]).max()


def test_c1_source_mode_lowrank_arnoldi_vs_reference():
    """C1: source mode (space-time parameter, low-rank in and out), Q1 32²,
    n_t 64, all nodes observed, prior (I + 0.1 L)⁻¹, r_max 20, low-rank
    Arnoldi m_a 10 from the reference's seeded rank-1 start."""
    ctx, grid, _ = _ctx(32, 2, "q1", 64, 0, 1, 0.01, 1.0, 0.1, 20, mode="source", full=True)
    fx = _fx("c1_source")
    v1 = lp.LowRankMat(fx["w1"].reshape(-1, 1), fx["w2"].reshape(-1, 1))
    res = lp.lr_arnoldi(ctx.apply, v1, ctx.pol, lp.StopRule(m_a=10, eps_eig=1e-1, check_every=10),
                        rank_source=ctx.rank_trace)
    assert res.iterations == int(fx["iters"][0])
    lead = fx["ritz"] >= 1e-1
    np.testing.assert_allclose(res.ritz_values.real[: lead.sum()], fx["ritz"][lead], rtol=1e-6)
    assert np.all(np.abs(np.array(res.rank_trace) - fx["ranks"]) <= 1), \
        (res.rank_trace, fx["ranks"].tolist())
    top = res.ritz_vectors[0]
    sv = lp.lr_singular_values(top)
    k = min(len(sv), len(fx["top_sv"]), 4)
    np.testing.assert_allclose(sv[:k], fx["top_sv"][:k], rtol=1e-5, atol=1e-9)


@pytest.mark.parametrize("form", ["auto", "persistent"])
def test_c4_path_3d_point_sensors_global_rows_vs_reference(monkeypatch, form):
    """The C4 path at n_x >= 1e5 (3-D 7-point heat 48³ = 110,592 dofs, rows
    not resident: the streaming-flush sweep by default, the persistent kernel's
    global-row phases with LRK_SFLUSH=0): 12³ point sensors every 4th step,
    σ 0.005, prior (I + 0.02 L)⁻¹, r_max 64 — one apply against the reference."""
    if form == "persistent":
        monkeypatch.setenv("LRK_SFLUSH", "0")
    ctx, grid, _ = _ctx(48, 3, "fd", 32, 12, 4, 0.005, 1.0, 0.02, 64)
    fx = _fx("c4_sweep3d")
    v = np.random.default_rng(3).standard_normal(grid.n_x)
    _check_apply(ctx, v / np.linalg.norm(v), fx)


@pytest.mark.parametrize("modes", [(1, 1, 1), (2, 1, 3)])
def test_c4_full_size_closed_form_eigenpair(modes):
    """C4 at FULL size (128³ = 2.1M dofs, n_t 2048, obs every 4th step,
    σ 0.005, prior (I + 0.02 L)⁻¹): DST-mode input gives μ v with
    μ = β τ M Σ_{k ≡ 0 mod 4} θ^{2k} (δ+γλ)⁻²."""
    ctx, grid, bn = _ctx(128, 3, "fd", 2048, 0, 4, 0.005, 1.0, 0.02, 64, full=True)
    v = O.config_eigvec(modes, 128)
    out = ctx.apply(v)
    mu = O.config_ic_eigenvalue(modes, 128, 2048, bn, 1.0, "fd", (1.0, 0.02), 4)
    assert np.linalg.norm(out - mu * v) <= 1e-8 * mu


def test_gmres_c1_size_vs_reference():
    """Device-resident factored GMRES (lrk_st_solve, LRK_SOLVE_GMRES) at the C1
    operator size (Q1 32², n_t 64): iterations within ±1 of the reference and
    the solution to its truncation tolerance, forward and adjoint."""
    fx = _fx("c1_gmres")
    grid = lp.build_grid(32)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid, "q1"), lp.build_time_grid(64))
    rhs = lp.LowRankMat(fx["R1"], fx["R2"])
    for tag, adj in (("f", False), ("b", True)):
        tr = []
        Y = lp.st_solve_krylov(K, rhs, lp.TruncationPolicy(), adjoint=adj, trace=tr)
        assert abs(len(tr) - len(fx[f"{tag}_trace"])) <= 1
        ref = fx[f"{tag}_Y1"] @ fx[f"{tag}_Y2"].T
        assert np.linalg.norm(lp.lr_to_dense(Y) - ref) <= 1e-7 * np.linalg.norm(ref)
        # and it solves the all-at-once system to the GMRES tolerance
        S = lp.st_solve_sweep(K, rhs, lp.TruncationPolicy(), adjoint=adj)
        assert np.linalg.norm(lp.lr_to_dense(Y) - lp.lr_to_dense(S)) <= \
            1e-6 * np.linalg.norm(lp.lr_to_dense(S))


def test_gmres_convergence_failure_carries_residual():
    grid = lp.build_grid(16, 2)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid, "q1"), lp.build_time_grid(32))
    rng = np.random.default_rng(5)
    rhs = lp.LowRankMat(rng.standard_normal((grid.n_x, 2)), rng.standard_normal((32, 2)))
    with pytest.raises(lp.ConvergenceFailure) as ei:
        lp.st_solve_krylov(K, rhs, lp.TruncationPolicy(), max_iter=3)
    assert ei.value.iterations == 3
    assert 0.0 < ei.value.achieved_residual < 1.0


# ------------------------------------------------ wide concatenations
def _sum_dense(terms, coefs):
    return sum(c * (t.W1.cpu().numpy() @ t.W2.cpu().numpy().T) for t, c in zip(terms, coefs))


@pytest.mark.parametrize("n_x,n_t,nterms,basis", [(2000, 100, 120, None), (90, 700, 110, None),
                                                   (500, 400, 120, 40)])
def test_add_truncate_wider_than_the_core(n_x, n_t, nterms, basis):
    """One truncation of a 240-column concatenation: short-side dense product
    (n_t or n_x <= 160) or rounding-floor folds (both long, low numerical
    rank) — against the oracle's truncation of the same sum."""
    rng = np.random.default_rng(n_x + n_t)
    if basis is None:
        terms = [lp.LowRankMat(rng.standard_normal((n_x, 2)) * 0.7 ** i,
                               rng.standard_normal((n_t, 2))) for i in range(nterms)]
    else:
        B1, B2 = rng.standard_normal((n_x, basis)), rng.standard_normal((n_t, basis))
        terms = [lp.LowRankMat(B1[:, rng.integers(0, basis, 2)], B2[:, rng.integers(0, basis, 2)])
                 for _ in range(nterms)]
    coefs = rng.standard_normal(nterms)
    pol = lp.TruncationPolicy(1e-8)
    out = lp.lr_add_truncate(terms, coefs, pol)
    A = _sum_dense(terms, coefs)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    r = O.rank_cut(s, 1e-8)
    assert out.r == r
    assert np.linalg.norm(lp.lr_to_dense(out) - A) <= 1e-8 * np.linalg.norm(A) * (1 + 1e-9)
    # the single-term wide path of lr_truncate (formerly an endless fold loop)
    big = lp.LowRankMat(np.hstack([t.W1.cpu().numpy() for t in terms]),
                        np.hstack([c * t.W2.cpu().numpy() for t, c in zip(terms, coefs)]))
    out2 = lp.lr_truncate(big, pol)
    assert out2.r == r


def test_wide_truncation_of_full_rank_input_fails_cleanly():
    X = np.random.default_rng(9).standard_normal((200, 200))
    with pytest.raises(NotImplementedError):
        lp.lr_from_dense(X, lp.TruncationPolicy(1e-8))
    Y = np.random.default_rng(9).standard_normal((200, 50)) @ np.random.default_rng(10).standard_normal((50, 200))
    out = lp.lr_from_dense(Y, lp.TruncationPolicy(1e-8))
    assert out.r == 50
    assert np.linalg.norm(lp.lr_to_dense(out) - Y) <= 1e-8 * np.linalg.norm(Y)


def test_sweep_core_overflow_is_reported_not_silent():
    """r_max beyond 160 - compress_every cannot fit the device core: the apply
    must raise instead of returning a silently truncated (zero) result."""
    grid = lp.build_grid(24)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(16))
    cov = lp.CovarianceSpec(1e6, 1.0, 1.0)
    ctx = lp.HessianContext(mode="ic", operator=K, layout=lp.full_observation(grid), cov=cov,
                            pol=lp.TruncationPolicy(1e-8, 150), compress_every=16)
    with pytest.raises(NotImplementedError):
        ctx.apply(np.ones(grid.n_x))


def test_batched_lr_dots_match_pairwise():
    from paper_1703_05638_b200.arnoldi import _FieldStore
    rng = np.random.default_rng(12)
    n_x, n_t = 3000, 70
    fields = [lp.LowRankMat(rng.standard_normal((n_x, r)), rng.standard_normal((n_t, r)))
              for r in (1, 5, 17, 3, 64, 2)]
    st = _FieldStore(n_x, n_t, cap=8)
    for f in fields:
        st.append(f)
    w = lp.LowRankMat(rng.standard_normal((n_x, 9)), rng.standard_normal((n_t, 9)))
    got = st.dots(w)
    ref = np.array([O.dot((w.W1.cpu().numpy(), w.W2.cpu().numpy()),
                          (f.W1.cpu().numpy(), f.W2.cpu().numpy())) for f in fields])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("name", ["hic_d", "cfg_q1b"])
def test_streaming_flush_small_fixtures_vs_reference(golden, monkeypatch, name):
    """The streaming-flush sweep forced on the reference's small rank-capped
    fixtures (ragged last chunk, tiny grids): same outputs and max ranks."""
    monkeypatch.setenv("LRK_SFLUSH", "1")
    if name == "hic_d":
        n_side, n_t, bn, bp, gp, rmax = golden["hic_d_meta"]
        grid = lp.build_grid(int(n_side))
        K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(int(n_t)))
        cov = lp.CovarianceSpec(bn, bp, gp)
        layout = lp.SensorLayout((), golden["hic_d_mask"])
        ctx = lp.HessianContext(mode="ic", operator=K, layout=layout, cov=cov,
                                pol=lp.TruncationPolicy(1e-8, int(rmax)))
    else:
        meta = golden["cfg_q1b_meta"]
        n_side, n_t, delta, gp, bn, rmax = int(meta[0]), int(meta[3]), meta[5], meta[6], meta[7], int(meta[8])
        grid = lp.build_grid(n_side)
        K = lp.SpaceTimeOperator(lp.assemble_heat(grid, "q1"), lp.build_time_grid(n_t))
        cov = lp.CovarianceSpec(bn, 1.0, 1.0, prior_delta=delta, prior_gamma=gp)
        ctx = lp.HessianContext(mode="ic", operator=K, layout=lp.SensorLayout((), golden["cfg_q1b_mask"]),
                                cov=cov, pol=lp.TruncationPolicy(1e-8, rmax))
    V, Oref = golden[f"{name}_V"], golden[f"{name}_O"]
    refr = golden[f"{name}_ranks"]
    for j in range(V.shape[1]):
        out = ctx.apply(V[:, j])
        assert np.linalg.norm(out - Oref[:, j]) <= 1e-9 * np.linalg.norm(Oref[:, j])
        if refr.size == V.shape[1]:
            assert ctx.rank_trace[-1] == refr[j]


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_nx_sharded_streaming_sweep_c4_path_vs_reference(shards):
    """The n_x-sharded streaming sweep — row slabs with their
    own partial tables, rank totals exchanged through the SFXBuf slots and
    release/acquire flags, one-CTA tail kernels — driven for all shards by one
    process (single-device emulation: the kernels and the exchange protocol
    are the ones the multi-process path runs over peer memory).  C4-path
    apply against the reference fixture: values and rank trace."""
    from paper_1703_05638_b200 import _lib

    ctx, grid, _ = _ctx(48, 3, "fd", 32, 12, 4, 0.005, 1.0, 0.02, 64)
    assert _lib.get_lib().lrk_set_emulated_shards(ctx._dev.handle, shards) == 0
    fx = _fx("c4_sweep3d")
    v = np.random.default_rng(3).standard_normal(grid.n_x)
    _check_apply(ctx, v / np.linalg.norm(v), fx)


def test_nx_sharded_streaming_sweep_c2_config_vs_unsharded(monkeypatch):
    """C2 bench configuration with the streaming form forced: 2 and 8 row
    shards against the unsharded streaming sweep — identical rank traces,
    values equal to rounding (the shard totals are summed in a different
    order than the CTA partials of one device)."""
    from paper_1703_05638_b200 import _lib

    monkeypatch.setenv("LRK_SFLUSH", "1")
    ctx, grid, _ = _c2()
    v = np.random.default_rng(1).standard_normal(grid.n_x)
    v /= np.linalg.norm(v)
    a = ctx.apply(v)
    tr_a = ctx.last_traces()
    for shards in (2, 8):
        assert _lib.get_lib().lrk_set_emulated_shards(ctx._dev.handle, shards) == 0
        b = ctx.apply(v)
        tr_b = ctx.last_traces()
        assert tr_a == tr_b
        np.testing.assert_allclose(b, a, rtol=0, atol=1e-11 * np.abs(a).max())


def test_shard_arena_world_one_c4_path_vs_reference():
    """lrk_shard_setup with a world of one: the sweep panes move into the
    IPC-exportable arena (the layout every rank of a sharded job uses) and the
    apply still reproduces the reference."""
    import ctypes

    from paper_1703_05638_b200 import _lib

    ctx, grid, _ = _ctx(48, 3, "fd", 32, 12, 4, 0.005, 1.0, 0.02, 64)
    h = ctypes.create_string_buffer(64)
    assert _lib.get_lib().lrk_shard_setup(ctx._dev.handle, 0, 1, h) == 0
    assert any(h.raw)
    assert _lib.get_lib().lrk_shard_connect(ctx._dev.handle, h) == 0
    fx = _fx("c4_sweep3d")
    v = np.random.default_rng(3).standard_normal(grid.n_x)
    _check_apply(ctx, v / np.linalg.norm(v), fx)


def test_streaming_flush_at_the_rank_cap_matches_persistent(monkeypatch):
    """Pane ranks up to the 64-column cap (72 staged columns per tile: the
    passes then stream with fewer warps so that two ring slots per warp still
    fit): the streaming-flush sweep against the persistent kernel on a
    full-rank forcing — identical rank traces, values to rounding."""
    rng = np.random.default_rng(77)
    n_side, n_t = 48, 96
    grid = lp.build_grid(n_side)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
    rhs = lp.LowRankMat(rng.standard_normal((grid.n_x, 40)), rng.standard_normal((n_t, 40)))
    pol = lp.TruncationPolicy(1e-13, 64)
    out = {}
    for form in ("0", "1"):
        monkeypatch.setenv("LRK_SFLUSH", form)
        tr = []
        Y = lp.st_solve_sweep(K, rhs, pol, trace=tr)
        out[form] = (tr, (Y.W1 @ Y.W2.T).cpu().numpy())
    assert max(out["1"][0]) == 64, out["1"][0]
    assert out["0"][0] == out["1"][0]
    ref = out["0"][1]
    assert np.abs(out["1"][1] - ref).max() <= 1e-10 * np.abs(ref).max()


@pytest.mark.parametrize("shards", [1, 4])
def test_streaming_sweep_is_bitwise_reproducible(shards):
    """Every reduction of the streaming-flush sweep runs in a fixed order (CTA
    partials by the last CTA, shard totals in shard order), so repeated applies
    of the same vector return the same bits — also with the generation running
    concurrently on the second stream."""
    from paper_1703_05638_b200 import _lib

    ctx, grid, _ = _ctx(48, 3, "fd", 32, 12, 4, 0.005, 1.0, 0.02, 64)
    if shards > 1:
        assert _lib.get_lib().lrk_set_emulated_shards(ctx._dev.handle, shards) == 0
    v = np.random.default_rng(5).standard_normal(grid.n_x)
    outs = [ctx.apply(v) for _ in range(3)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


@pytest.mark.parametrize("form", ["0", "1"], ids=["persistent", "streaming"])
@pytest.mark.parametrize("n_side,dim,n_t,r_max,sensors", [
    (5, 2, 1, None, "full"),      # a single time step: one ragged flush of one column
    (7, 2, 3, None, "full"),      # fewer steps than one flush
    (11, 2, 6, 1, "sub"),         # n_x = 121 (cuts the 8-row tiles), rank cap 1
    (9, 2, 10, 3, "none"),        # no sensors: the observation field is zero
    (5, 3, 7, None, "sub"),       # 3-D, n_x = 125, ragged last flush
    (6, 3, 9, 2, "full"),         # 3-D, n_x = 216, tight cap
])
def test_sweep_forms_on_ragged_and_degenerate_shapes_vs_oracle(monkeypatch, form, n_side, dim, n_t,
                                                               r_max, sensors):
    """Edge shapes through both sweep forms (rows resident / streaming flushes) against the
    oracle: ragged flushes (n_t not a multiple of compress_every), row counts that cut the
    8-row tiles, rank caps of 1-3, an empty sensor set, and the zero vector."""
    monkeypatch.setenv("LRK_SFLUSH", form)
    grid = lp.build_grid(n_side, dim)
    K = lp.SpaceTimeOperator(lp.assemble_heat(grid), lp.build_time_grid(n_t))
    rng = np.random.default_rng(1000 + 37 * n_side + n_t)
    if sensors == "full":
        mask = np.ones(grid.n_x, dtype=bool)
    elif sensors == "none":
        mask = np.zeros(grid.n_x, dtype=bool)
    else:
        mask = rng.random(grid.n_x) < 0.3
    bn = 1.0 / (0.02**2 * K.time.tau * grid.m_scale)
    cov = lp.CovarianceSpec(bn, 1.0, 1.0)
    ctx = lp.HessianContext(mode="ic", operator=K, layout=lp.SensorLayout((), mask), cov=cov,
                            pol=lp.TruncationPolicy(1e-8, r_max))
    P = O.Problem(n_side, n_t, mask, bn, 1.0, 1e-8, r_max, dim=dim)
    assert np.count_nonzero(ctx.apply(np.zeros(grid.n_x))) == 0
    for _ in range(2):
        v = rng.standard_normal(grid.n_x)
        ref, rank = O.hessian_ic(P, v)
        got = ctx.apply(v)
        scale = np.linalg.norm(ref)
        if scale == 0.0:
            assert np.count_nonzero(got) == 0
        else:
            assert np.linalg.norm(got - ref) <= 1e-9 * scale
        assert ctx.rank_trace[-1] == rank
