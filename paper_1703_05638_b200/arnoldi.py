"""Low-rank Arnoldi with full reorthogonalisation (mirrors lrpostcov/arnoldi.py).

Algorithm 1 of the paper as the reference implements it (arnoldi.py:271-375):
apply, two orthogonalisation passes accumulating ``H[i, j] +=``, breakdown
at 1e-14 (stop or seeded restart), Ritz refresh every ``check_every``.
Dense (IC/steady) iterates live in one device matrix and are orthogonalised
with a two-pass classical Gram-Schmidt in liblrk.so (lrk_cgs2 — the CGS2 form
of the reference's MGS2, identical in exact arithmetic); low-rank iterates
use the device lr_* operations with the reference's work_cap=48 policy.  The
k x k Hessenberg eigenproblems stay on the host in numpy, exactly as in the
reference, so Ritz values are computed by the same LAPACK routine.
"""

from __future__ import annotations

import time as _time
from ctypes import byref, c_double
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NumericalError
from .lowrank import (
    LowRankMat,
    TruncationPolicy,
    colmajor,
    lr_add,
    lr_dot,
    lr_norm,
    lr_scale,
    lr_singular_values,
    lr_truncate,
)

BREAKDOWN_TOL = 1e-14


@dataclass(frozen=True)
class StopRule:
    """Iteration cap plus eigenvalue-threshold stopping (arnoldi.py:38-62)."""

    m_a: int
    eps_eig: float = 1e-1
    check_every: int = 10
    stability_rtol: float = 1e-3
    on_breakdown: str = "stop"
    restart_seed: int = 0

    def __post_init__(self):
        if self.m_a < 1:
            raise ValueError(f"m_a must be >= 1, got {self.m_a}")
        if self.eps_eig <= 0:
            raise ValueError(f"eps_eig must be positive, got {self.eps_eig}")
        if self.on_breakdown not in ("stop", "restart"):
            raise ValueError(f"on_breakdown must be stop or restart, got {self.on_breakdown!r}")


@dataclass
class ArnoldiResult:
    H: np.ndarray
    basis: list
    rank_trace: list
    ritz_values: np.ndarray
    ritz_vectors: list
    converged_count: int
    breakdown: bool
    iterations: int
    diagnostics: list
    restarts: int = 0

    def gram_defect(self) -> float:
        """max |<v_i, v_j> - δ_ij| over the stored basis."""
        ops = _ops_for(self.basis[0])
        worst = 0.0
        for i in range(len(self.basis)):
            for j in range(i, len(self.basis)):
                g = ops.dot(self.basis[i], self.basis[j])
                worst = max(worst, abs(g - (1.0 if i == j else 0.0)))
        return worst


def _torch():
    import torch

    return torch


class _DenseOps:
    """Dense spatial vectors (numpy or device tensors)."""

    def __init__(self, pol: TruncationPolicy):
        self.pol = pol

    @staticmethod
    def dot(a, b) -> float:
        if isinstance(a, np.ndarray) and isinstance(b, np.ndarray):
            return float(np.dot(a, b))
        torch = _torch()
        return float(torch.dot(torch.as_tensor(a, device="cuda", dtype=torch.float64).reshape(-1),
                               torch.as_tensor(b, device="cuda", dtype=torch.float64).reshape(-1)))

    @staticmethod
    def norm(a) -> float:
        return float(np.sqrt(max(_DenseOps.dot(a, a), 0.0)))

    @staticmethod
    def scale(a, c):
        return a * c

    @staticmethod
    def rank(w) -> int:
        return 0


class _LowRankOps:
    """LowRankMat iterates with working-rank control (arnoldi.py:128-166)."""

    def __init__(self, pol: TruncationPolicy, work_cap: int = 48):
        self.pol = pol
        self.work_cap = work_cap

    @staticmethod
    def dot(a, b) -> float:
        return lr_dot(a, b)

    @staticmethod
    def norm(a) -> float:
        return lr_norm(a)

    @staticmethod
    def scale(a, c):
        return lr_scale(a, c)

    def sub(self, w, h, v):
        w = lr_add(w, lr_scale(v, -h))
        if w.r > self.work_cap:
            w = lr_truncate(w, self.pol)
        return w

    def compress(self, w, final=False):
        return lr_truncate(w, self.pol)

    @staticmethod
    def rank(w) -> int:
        return w.r

    def combine(self, basis, coeffs):
        out = LowRankMat.zeros(*basis[0].shape)
        for v, c in zip(basis, coeffs):
            out = lr_add(out, lr_scale(v, float(np.real(c))))
            if out.r > self.work_cap:
                out = lr_truncate(out, self.pol)
        return lr_truncate(out, self.pol)


def _ops_for(v, pol: TruncationPolicy | None = None):
    pol = pol or TruncationPolicy()
    return _LowRankOps(pol) if isinstance(v, LowRankMat) else _DenseOps(pol)


def _hessenberg_eigs(Hm: np.ndarray):
    try:
        vals, vecs = np.linalg.eig(Hm)
    except np.linalg.LinAlgError as exc:
        raise NumericalError(f"dense Hessenberg eigensolve failed: {exc}") from exc
    order = np.argsort(-vals.real)
    return vals[order], vecs[:, order]


def _coeffs(H: np.ndarray):
    """Ritz values and combination coefficients (arnoldi.py:197-204)."""
    m = H.shape[1]
    Hm = H[:m, :m]
    vals, vecs = _hessenberg_eigs(Hm)
    scale = float(np.abs(Hm).max()) if m else 0.0
    defect = float(np.abs(Hm - Hm.T).max()) if m else 0.0
    if scale > 0 and defect <= 1e-6 * scale:
        _, sym_vecs = np.linalg.eigh(0.5 * (Hm + Hm.T))
        vecs = sym_vecs[:, ::-1]
    return vals, vecs


class _DenseBasis:
    """Arnoldi basis held as columns of one device matrix."""

    def __init__(self, n: int, cap: int, as_numpy: bool):
        self.Q = colmajor(n, cap)
        self.n = n
        self.k = 0
        self.as_numpy = as_numpy
        self._ctx = _lib.algebra_context()

    def push(self, v_dev):
        self.Q[:, self.k] = v_dev
        self.k += 1

    def user(self, i):
        col = self.Q[:, i]
        return col.cpu().numpy() if self.as_numpy else col

    def cgs2(self, w_dev, k):
        h = (c_double * max(k, 1))()
        nrm = c_double(0.0)
        _lib.check(
            _lib.get_lib().lrk_cgs2(self._ctx.handle, self.Q.data_ptr(), self.n, k,
                                    w_dev.data_ptr(), self.n, h, byref(nrm), _lib.stream_handle()),
            self._ctx.handle, "lr_arnoldi")
        return np.array(h[:k]), float(nrm.value)

    def combine(self, coeffs):
        torch = _torch()
        k = len(coeffs)
        y = torch.empty(self.n, dtype=torch.float64, device=self.Q.device)
        cf = (c_double * max(k, 1))(*[float(np.real(c)) for c in coeffs])
        _lib.check(
            _lib.get_lib().lrk_combine(self._ctx.handle, self.Q.data_ptr(), self.n, k, cf, self.n,
                                       y.data_ptr(), _lib.stream_handle()),
            self._ctx.handle, "ritz_pairs")
        return y


def _to_dev_vec(x):
    torch = _torch()
    return torch.as_tensor(np.asarray(x) if isinstance(x, np.ndarray) else x,
                           dtype=torch.float64).reshape(-1).to("cuda").contiguous()


def ritz_pairs(H: np.ndarray, basis: list, pol: TruncationPolicy | None = None) -> list:
    """Ritz pairs from the leading m x m block (arnoldi.py:184-213)."""
    m = H.shape[1]
    vals, vecs = _coeffs(H)
    if isinstance(basis[0], LowRankMat):
        ops = _LowRankOps(pol or TruncationPolicy())
        pairs = []
        for i in range(m):
            v = ops.combine(basis[:m], vecs[:, i])
            nrm = ops.norm(v)
            if nrm > 0:
                v = ops.scale(v, 1.0 / nrm)
            pairs.append((complex(vals[i]), v))
        return pairs
    as_np = isinstance(basis[0], np.ndarray)
    n = int(np.asarray(basis[0]).shape[0]) if as_np else int(basis[0].shape[0])
    B = _DenseBasis(n, m, as_np)
    for i in range(m):
        B.push(_to_dev_vec(basis[i]))
    pairs = []
    for i in range(m):
        y = B.combine(vecs[:, i])
        nrm = float(y.norm())
        if nrm > 0:
            y = y / nrm
        pairs.append((complex(vals[i]), y.cpu().numpy() if as_np else y))
    return pairs


def _stop_ready(vals, prev, stop: StopRule):
    """Refresh-to-refresh stopping condition (arnoldi.py:242-268)."""
    above = int(np.sum(vals.real >= stop.eps_eig))
    if prev is None:
        return False, above
    if above != int(np.sum(prev.real >= stop.eps_eig)):
        return False, above
    n_check = above if above > 0 else min(1, len(vals), len(prev))
    if n_check > len(prev):
        return False, above
    for i in range(n_check):
        denom = max(abs(vals[i].real), abs(prev[i].real), 1e-300)
        if abs(vals[i].real - prev[i].real) / denom > stop.stability_rtol:
            return False, above
    return True, above


def _fresh_lowrank(basis, ops, seed):
    rng = np.random.default_rng(0x5EED + seed)
    n_x, n_t = basis[0].shape
    w = LowRankMat(rng.standard_normal((n_x, 2)), rng.standard_normal((n_t, 2)))
    w = ops.scale(w, 1.0 / ops.norm(w))
    for _pass in range(2):
        for v in basis:
            w = ops.sub(w, ops.dot(w, v), v)
        w = ops.compress(w)
    nrm = ops.norm(w)
    if nrm <= 1e-6:
        return None
    return ops.compress(ops.scale(w, 1.0 / nrm))


def lr_arnoldi(apply, v1, pol: TruncationPolicy, stop: StopRule,
               rank_source: list | None = None) -> ArnoldiResult:
    """Arnoldi iteration for a self-adjoint-up-to-truncation operator (arnoldi.py:271-375)."""
    if isinstance(v1, LowRankMat):
        return _arnoldi_lowrank(apply, v1, pol, stop, rank_source)
    return _arnoldi_dense(apply, v1, pol, stop, rank_source)


def _finish(H, j_done, basis_user, pol, stop, prev_vals, rank_trace, diagnostics, breakdown,
            restarts):
    Hout = H[: j_done + 1, : j_done]
    pairs = ritz_pairs(Hout, basis_user, pol)
    vals = np.array([p[0] for p in pairs])
    if prev_vals is not None:
        _, converged = _stop_ready(vals, prev_vals, stop)
    else:
        converged = int(np.sum(vals.real >= stop.eps_eig))
    return ArnoldiResult(H=Hout, basis=basis_user, rank_trace=rank_trace, ritz_values=vals,
                         ritz_vectors=[p[1] for p in pairs], converged_count=converged,
                         breakdown=breakdown, iterations=j_done, diagnostics=diagnostics,
                         restarts=restarts)


def _arnoldi_dense(apply, v1, pol, stop, rank_source):
    as_np = isinstance(v1, np.ndarray) or not _torch().is_tensor(v1)
    v = _to_dev_vec(v1)
    nrm = float(v.norm())
    if nrm == 0:
        raise ValueError("start vector must be nonzero")
    n = v.numel()
    B = _DenseBasis(n, stop.m_a + 1, as_np)
    B.push(v / nrm)
    H = np.zeros((stop.m_a + 1, stop.m_a))
    rank_trace, diagnostics = [], []
    prev_vals, breakdown, restarts, j_done = None, False, 0, 0
    src_seen = len(rank_source) if rank_source is not None else 0
    for j in range(stop.m_a):
        t0 = _time.perf_counter()
        w = _to_dev_vec(apply(B.user(j))).clone()
        apply_rank = 0
        if rank_source is not None and len(rank_source) > src_seen:
            apply_rank = max(rank_source[src_seen:])
            src_seen = len(rank_source)
        h, h_sub = B.cgs2(w, B.k)
        H[: B.k, j] += h
        H[j + 1, j] = h_sub
        rank_trace.append(apply_rank)
        diagnostics.append((j + 1, h_sub, apply_rank, _time.perf_counter() - t0))
        j_done = j + 1
        if h_sub <= BREAKDOWN_TOL:
            breakdown = True
            if stop.on_breakdown != "restart" or j + 1 >= stop.m_a:
                break
            H[j + 1, j] = 0.0
            rng = np.random.default_rng(0x5EED + stop.restart_seed + restarts)
            f = _to_dev_vec(rng.standard_normal(n))
            f = f / float(f.norm())
            _, fn = B.cgs2(f, B.k)
            if fn <= 1e-6:
                break
            restarts += 1
            B.push(f / fn)
            continue
        B.push(w / h_sub)
        if (j + 1) % stop.check_every == 0 and j + 1 < stop.m_a:
            vals, _ = _hessenberg_eigs(H[: j + 1, : j + 1])
            ready, _ = _stop_ready(vals, prev_vals, stop)
            prev_vals = vals
            if ready:
                break
    basis_user = [B.user(i) for i in range(B.k)]
    return _finish(H, j_done, basis_user, pol, stop, prev_vals, rank_trace, diagnostics,
                   breakdown, restarts)


def _arnoldi_lowrank(apply, v1, pol, stop, rank_source):
    ops = _LowRankOps(pol)
    nrm = ops.norm(v1)
    if nrm == 0:
        raise ValueError("start vector must be nonzero")
    basis = [ops.compress(ops.scale(v1, 1.0 / nrm))]
    H = np.zeros((stop.m_a + 1, stop.m_a))
    rank_trace, diagnostics = [], []
    prev_vals, breakdown, restarts, j_done = None, False, 0, 0
    src_seen = len(rank_source) if rank_source is not None else 0
    for j in range(stop.m_a):
        t0 = _time.perf_counter()
        w = apply(basis[j])
        apply_rank = ops.rank(w)
        if rank_source is not None and len(rank_source) > src_seen:
            apply_rank = max(apply_rank, max(rank_source[src_seen:]))
            src_seen = len(rank_source)
        for _pass in range(2):
            for i in range(j + 1):
                hij = ops.dot(w, basis[i])
                H[i, j] += hij
                w = ops.sub(w, hij, basis[i])
            w = ops.compress(w)
        h_sub = ops.norm(w)
        H[j + 1, j] = h_sub
        max_rank = max(apply_rank, ops.rank(w))
        rank_trace.append(max_rank)
        diagnostics.append((j + 1, h_sub, max_rank, _time.perf_counter() - t0))
        j_done = j + 1
        if h_sub <= BREAKDOWN_TOL:
            breakdown = True
            if stop.on_breakdown != "restart" or j + 1 >= stop.m_a:
                break
            H[j + 1, j] = 0.0
            fresh = _fresh_lowrank(basis, ops, stop.restart_seed + restarts)
            if fresh is None:
                break
            restarts += 1
            basis.append(fresh)
            continue
        basis.append(ops.compress(ops.scale(w, 1.0 / h_sub)))
        if (j + 1) % stop.check_every == 0 and j + 1 < stop.m_a:
            vals, _ = _hessenberg_eigs(H[: j + 1, : j + 1])
            ready, _ = _stop_ready(vals, prev_vals, stop)
            prev_vals = vals
            if ready:
                break
    return _finish(H, j_done, basis, pol, stop, prev_vals, rank_trace, diagnostics, breakdown,
                   restarts)


def rank_one_check(vec, reshape=None, tail_tol: float = 1e-6):
    """Numerical separation rank of a vector (arnoldi.py:378-399); diagnostic."""
    if isinstance(vec, LowRankMat):
        s = lr_singular_values(vec)
    else:
        if reshape is None:
            raise ValueError("dense input needs an explicit 2-way reshape")
        torch = _torch()
        X = torch.as_tensor(np.asarray(vec) if isinstance(vec, np.ndarray) else vec,
                            dtype=torch.float64).reshape(reshape)
        s = torch.linalg.svdvals(X.to("cuda")).cpu().numpy()
    if s.size == 0 or s[0] == 0.0:
        return 0, 0.0
    total = float(np.linalg.norm(s))
    tail = np.sqrt(np.cumsum(s[::-1] ** 2))[::-1]
    r = int(np.searchsorted(-tail, -tail_tol * total, side="left"))
    return r, (float(s[1] / s[0]) if s.size > 1 else 0.0)
