"""Arnoldi recurrence around the Hessian apply, with its Krylov basis on the device.

Drop-in for lrpostcov.arnoldi (arnoldi.py:271-375): same public names
(StopRule, ArnoldiResult, lr_arnoldi, ritz_pairs, rank_one_check), same
stopping rule, breakdown/restart behaviour and Ritz extraction; Algorithm 1
of the paper.

The recurrence itself is organised around a *Krylov space* object that owns
the basis on the device and performs one full re-orthogonalised step per call:

* dense iterates (IC / steady parameters): the basis is the column block of one
  device matrix; each orthogonalisation pass is one `lrk_cgs2` call (batched
  Gram of w against every basis column, subtraction, one readback);
* low-rank iterates (space-time source parameter): the basis fields are stored
  as contiguous column ranges of one n_x x C and one n_t x C device matrix.
  A pass evaluates every inner product <w, V_i> with ONE batched Gram
  (`lrk_lr_dots`) and turns them into the reference's *modified* Gram-Schmidt
  coefficients with the basis Gram G_li = <V_l, V_i> (kept current, one batched
  dot per new field): h_i = c_i - sum_{l<i} h_l G_li, which is MGS exactly in
  exact arithmetic because the subtraction is an exact concatenation.  The
  subtraction then costs one fused concatenate-and-truncate
  (`lrk_add_truncate`) per segment between the reference's work_cap = 48
  truncations (arnoldi.py:141-151), which are kept: a new batched Gram is
  taken after each such truncation, so the iterates follow the reference's.

The k x k Hessenberg eigenproblems stay on the host (numpy LAPACK, like the
reference), so Ritz values come from the same routine.
"""

from __future__ import annotations

import time as _time
from ctypes import byref, c_double, c_int
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NumericalError
from .lowrank import (
    LowRankMat,
    TruncationPolicy,
    colmajor,
    lr_add_truncate,
    lr_dot,
    lr_scale,
    lr_singular_values,
    lr_truncate,
)

BREAKDOWN_TOL = 1e-14   # arnoldi.py:35
WORK_CAP = 48           # working-rank cap of low-rank iterates (arnoldi.py:131)
RESTART_SALT = 0x5EED   # seed offset of restart directions (arnoldi.py:224)


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
    """Outcome of lr_arnoldi (arnoldi.py:65-87)."""

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
        """max |<v_i, v_j> - δ_ij| over the stored basis (batched on the device)."""
        G = _gram_matrix(self.basis)
        return float(np.abs(G - np.eye(G.shape[0])).max()) if G.size else 0.0


def _torch():
    import torch

    _lib.require_cuda()
    return torch


def _to_dev_vec(x):
    torch = _torch()
    return torch.as_tensor(np.asarray(x) if isinstance(x, np.ndarray) else x,
                           dtype=torch.float64).reshape(-1).to("cuda").contiguous()


# ----------------------------------------------------------------- dense space
class _DenseSpace:
    """Dense spatial iterates as columns of one device matrix; CGS2 on the device."""

    lowrank = False

    def __init__(self, v1, capacity: int):
        self.as_numpy = isinstance(v1, np.ndarray) or not _torch().is_tensor(v1)
        v = _to_dev_vec(v1)
        nrm = float(v.norm())
        if nrm == 0:
            raise ValueError("start vector must be nonzero")
        self.n = v.numel()
        self.Q = colmajor(self.n, capacity)
        self.k = 0
        self._ctx = _lib.algebra_context()
        self._push(v / nrm)

    def _push(self, v):
        if self.k == self.Q.shape[1]:  # restarts can exceed the planned size
            Q = colmajor(self.n, 2 * self.k)
            Q[:, : self.k] = self.Q[:, : self.k]
            self.Q = Q
        self.Q[:, self.k] = v
        self.k += 1

    def current(self):
        col = self.Q[:, self.k - 1]
        return col.cpu().numpy() if self.as_numpy else col

    def prepare(self, w):
        return _to_dev_vec(w).clone()

    def orthogonalize(self, w):
        """Two CGS passes against all k columns: (h, ||w||, w)."""
        k = self.k
        h = (c_double * max(k, 1))()
        nrm = c_double(0.0)
        _lib.check(
            _lib.get_lib().lrk_cgs2(self._ctx.handle, self.Q.data_ptr(), self.n, k, w.data_ptr(),
                                    self.n, h, byref(nrm), _lib.stream_handle()),
            self._ctx.handle, "lr_arnoldi")
        return np.array(h[:k]), float(nrm.value), w

    def extend(self, w, h_sub):
        self._push(w / h_sub)

    def fresh(self, seed):
        rng = np.random.default_rng(RESTART_SALT + seed)
        f = _to_dev_vec(rng.standard_normal(self.n))
        f = f / float(f.norm())
        _, fn, f = self.orthogonalize(f)
        if fn <= 1e-6:
            return None
        return f / fn

    def push_fresh(self, f):
        self._push(f)

    @staticmethod
    def rank(w) -> int:
        return 0

    def export(self) -> list:
        cols = [self.Q[:, i] for i in range(self.k)]
        return [c.cpu().numpy() for c in cols] if self.as_numpy else cols


# ------------------------------------------------------------- low-rank space
class _FieldStore:
    """Low-rank fields as contiguous column ranges of one n_x x C and one
    n_t x C device matrix, with batched inner products against all of them."""

    def __init__(self, n_x: int, n_t: int, cap: int = 64):
        self.n_x, self.n_t = n_x, n_t
        self._ctx = _lib.algebra_context()
        self.W1 = colmajor(n_x, cap)
        self.W2 = colmajor(n_t, cap)
        self.used = 0
        self.off, self.rk = [], []

    def __len__(self) -> int:
        return len(self.rk)

    def append(self, v: LowRankMat):
        if self.used + v.r > self.W1.shape[1]:
            cap = max(2 * self.W1.shape[1], self.used + v.r)
            W1, W2 = colmajor(self.n_x, cap), colmajor(self.n_t, cap)
            W1[:, : self.used] = self.W1[:, : self.used]
            W2[:, : self.used] = self.W2[:, : self.used]
            self.W1, self.W2 = W1, W2
        a = self.used
        self.W1[:, a:a + v.r] = v.W1
        self.W2[:, a:a + v.r] = v.W2
        self.off.append(a)
        self.rk.append(v.r)
        self.used += v.r

    def field(self, i: int) -> LowRankMat:
        a, r = self.off[i], self.rk[i]
        return LowRankMat._wrap(self.W1[:, a:a + r], self.W2[:, a:a + r])

    def dots(self, w: LowRankMat, k: int | None = None, lo: int = 0) -> np.ndarray:
        """<w, V_i> for fields lo <= i < k: one batched Gram + one readback."""
        k = len(self) if k is None else k
        if k <= lo:
            return np.zeros(0)
        nseg = k - lo
        out = (c_double * nseg)()
        seg = (c_int * nseg)(*self.rk[lo:k])
        a = self.off[lo]
        basis = LowRankMat._wrap(self.W1[:, a: self.used], self.W2[:, a: self.used])._c()
        _lib.check(
            _lib.get_lib().lrk_lr_dots(self._ctx.handle, byref(w._c()), byref(basis), nseg, seg,
                                       out, _lib.stream_handle()),
            self._ctx.handle, "lr_arnoldi")
        return np.array(out[:nseg])


def _lr_norm(w: LowRankMat) -> float:
    return float(np.sqrt(max(lr_dot(w, w), 0.0))) if w.r else 0.0


class _LowRankSpace:
    """Low-rank iterates in a _FieldStore plus their Gram matrix (see module doc)."""

    lowrank = True

    def __init__(self, v1: LowRankMat, pol: TruncationPolicy):
        self.pol = pol
        self.store = _FieldStore(*v1.shape)
        self.G = np.zeros((0, 0))
        nrm = _lr_norm(v1)
        if nrm == 0:
            raise ValueError("start vector must be nonzero")
        self._append(lr_truncate(lr_scale(v1, 1.0 / nrm), pol))

    def _append(self, v: LowRankMat):
        self.store.append(v)
        k = len(self.store)
        row = self.store.dots(self.store.field(k - 1))
        G = np.zeros((k, k))
        G[: k - 1, : k - 1] = self.G
        G[k - 1, :], G[:, k - 1] = row, row
        self.G = G

    @property
    def k(self) -> int:
        return len(self.store)

    def current(self) -> LowRankMat:
        return self.store.field(self.k - 1)

    def prepare(self, w):
        return w

    def _pass(self, w: LowRankMat):
        """One MGS pass of arnoldi.py:322-327 with its working-rank control
        (_LowRankOps.sub, arnoldi.py:141-151): the subtractions are exact
        concatenations, truncated whenever the working rank passes work_cap,
        and once more at the end of the pass (compress).  Between two
        truncations w is fixed up to the concatenated terms, so every MGS
        coefficient of the segment follows from ONE batched Gram against the
        segment's fields and the basis Gram: h_j = <w, V_j> - sum h_l <V_l, V_j>."""
        k = self.k
        h = np.zeros(k)
        i = 0
        while i < k:
            c = self.store.dots(w, k, lo=i)
            terms, coefs, width, j = [w], [1.0], w.r, i
            while j < k:
                h[j] = c[j - i] - h[i:j] @ self.G[i:j, j]
                if h[j] != 0.0:  # lr_scale by 0 is the zero field (lowrank.py:157-160)
                    terms.append(self.store.field(j))
                    coefs.append(-h[j])
                    width += self.store.rk[j]
                j += 1
                if width > WORK_CAP:
                    break
            w = lr_add_truncate(terms, coefs, self.pol)
            i = j
        if k == 0:
            w = lr_truncate(w, self.pol)
        return h, w

    def orthogonalize(self, w: LowRankMat):
        h1, w = self._pass(w)
        h2, w = self._pass(w)
        return h1 + h2, _lr_norm(w), w

    def extend(self, w: LowRankMat, h_sub: float):
        self._append(lr_scale(w, 1.0 / h_sub))

    def fresh(self, seed):
        rng = np.random.default_rng(RESTART_SALT + seed)
        n_x, n_t = self.store.n_x, self.store.n_t
        w = LowRankMat(rng.standard_normal((n_x, 2)), rng.standard_normal((n_t, 2)))
        w = lr_scale(w, 1.0 / _lr_norm(w))
        _, nrm, w = self.orthogonalize(w)
        if nrm <= 1e-6:
            return None
        return lr_truncate(lr_scale(w, 1.0 / nrm), self.pol)

    def push_fresh(self, f):
        self._append(f)

    @staticmethod
    def rank(w) -> int:
        return w.r

    def export(self) -> list:
        return [self.store.field(i) for i in range(self.k)]


# ------------------------------------------------------------ Ritz extraction
def _hessenberg_eigs(Hm: np.ndarray):
    """Eigenpairs of the leading square block, descending real part (arnoldi.py:174-181)."""
    try:
        vals, vecs = np.linalg.eig(Hm)
    except np.linalg.LinAlgError as exc:
        raise NumericalError(f"dense Hessenberg eigensolve failed: {exc}") from exc
    order = np.argsort(-vals.real)
    return vals[order], vecs[:, order]


def _ritz_coefficients(H: np.ndarray):
    """Ritz values and combination coefficients (arnoldi.py:197-204): the
    symmetric eigensolver's vectors when H_m is symmetric to 1e-6."""
    m = H.shape[1]
    Hm = H[:m, :m]
    vals, vecs = _hessenberg_eigs(Hm)
    if m:
        scale = float(np.abs(Hm).max())
        if scale > 0 and float(np.abs(Hm - Hm.T).max()) <= 1e-6 * scale:
            vecs = np.linalg.eigh(0.5 * (Hm + Hm.T))[1][:, ::-1]
    return vals, vecs


def _combine_dense(basis: list, coeffs: np.ndarray):
    """All Ritz vectors as one device product basis @ coeffs, columns normalised."""
    torch = _torch()
    Q = torch.stack([_to_dev_vec(b) for b in basis], dim=1)
    # a fresh copy: a 1 x 1 slice of a reversed array keeps its negative stride through
    # ascontiguousarray, which torch refuses
    Y = Q @ torch.as_tensor(np.array(np.real(coeffs), dtype=float, order="C"), dtype=torch.float64,
                             device=Q.device)
    nrm = Y.norm(dim=0)
    return Y / torch.where(nrm > 0, nrm, torch.ones_like(nrm))


def _combine_lowrank(basis: list, coeffs, pol: TruncationPolicy) -> LowRankMat:
    """sum_i c_i V_i with the reference's working-rank control (arnoldi.py:158-166):
    fused concatenate-and-truncate whenever the running width passes work_cap,
    and a final truncation."""
    out, i, k = None, 0, len(basis)
    while i < k:
        terms = [] if out is None else [out]
        cf = [] if out is None else [1.0]
        width = 0 if out is None else out.r
        while i < k:
            if float(coeffs[i]) != 0.0:
                terms.append(basis[i])
                cf.append(float(coeffs[i]))
                width += basis[i].r
            i += 1
            if width > WORK_CAP:
                break
        out = lr_add_truncate(terms, cf, pol) if terms else LowRankMat.zeros(*basis[0].shape)
    return out if out is not None else LowRankMat.zeros(*basis[0].shape)


def ritz_pairs(H: np.ndarray, basis: list, pol: TruncationPolicy | None = None) -> list:
    """Ritz pairs from the leading m x m block (arnoldi.py:184-213)."""
    m = H.shape[1]
    vals, vecs = _ritz_coefficients(H)
    if m == 0:
        return []
    if isinstance(basis[0], LowRankMat):
        pol = pol or TruncationPolicy()
        pairs = []
        for i in range(m):
            v = _combine_lowrank(basis[:m], np.real(vecs[:, i]), pol)
            nrm = _lr_norm(v)
            pairs.append((complex(vals[i]), lr_scale(v, 1.0 / nrm) if nrm > 0 else v))
        return pairs
    as_np = isinstance(basis[0], np.ndarray)
    Y = _combine_dense(basis[:m], vecs)
    cols = [Y[:, i] for i in range(m)]
    if as_np:
        Yh = Y.cpu().numpy()
        cols = [Yh[:, i] for i in range(m)]
    return [(complex(vals[i]), cols[i]) for i in range(m)]


def _gram_matrix(basis: list) -> np.ndarray:
    k = len(basis)
    if k == 0:
        return np.zeros((0, 0))
    if isinstance(basis[0], LowRankMat):
        st = _FieldStore(*basis[0].shape, cap=max(sum(b.r for b in basis), 1))
        for b in basis:
            st.append(b)
        return np.array([st.dots(st.field(i)) for i in range(k)])
    torch = _torch()
    Q = torch.stack([_to_dev_vec(b) for b in basis], dim=1)
    return (Q.T @ Q).cpu().numpy()


# --------------------------------------------------------------- stop rule
def _stop_ready(vals, prev, stop: StopRule):
    """(stop?, #values >= eps_eig) from two consecutive refreshes (arnoldi.py:242-268):
    same count above the threshold, and those leading values (or the leading
    one when none is above) stable to stability_rtol."""
    re = np.asarray(vals).real
    above = int(np.count_nonzero(re >= stop.eps_eig))
    if prev is None:
        return False, above
    pr = np.asarray(prev).real
    if above != int(np.count_nonzero(pr >= stop.eps_eig)):
        return False, above
    n = above if above else min(1, re.size, pr.size)
    if n > pr.size:
        return False, above
    a, b = re[:n], pr[:n]
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    return bool(np.all(np.abs(a - b) / denom <= stop.stability_rtol)), above


# --------------------------------------------------------------- the driver
def lr_arnoldi(apply, v1, pol: TruncationPolicy, stop: StopRule,
               rank_source: list | None = None) -> ArnoldiResult:
    """Arnoldi iteration for a self-adjoint-up-to-truncation operator (arnoldi.py:271-375)."""
    space = (_LowRankSpace(v1, pol) if isinstance(v1, LowRankMat)
             else _DenseSpace(v1, stop.m_a + 1))
    H = np.zeros((stop.m_a + 1, stop.m_a))
    ranks, diagnostics = [], []
    prev = None
    breakdown, restarts, done = False, 0, 0
    seen = len(rank_source) if rank_source is not None else 0
    for j in range(stop.m_a):
        t0 = _time.perf_counter()
        w = space.prepare(apply(space.current()))
        r_apply = space.rank(w)
        if rank_source is not None and len(rank_source) > seen:
            r_apply = max(r_apply, max(rank_source[seen:]))
            seen = len(rank_source)
        h, h_sub, w = space.orthogonalize(w)
        H[: h.size, j] += h
        H[j + 1, j] = h_sub
        r_step = max(r_apply, space.rank(w))
        ranks.append(r_step)
        diagnostics.append((j + 1, h_sub, r_step, _time.perf_counter() - t0))
        done = j + 1
        if h_sub <= BREAKDOWN_TOL:  # invariant subspace reached
            breakdown = True
            if stop.on_breakdown != "restart" or done >= stop.m_a:
                break
            H[j + 1, j] = 0.0
            f = space.fresh(stop.restart_seed + restarts)
            if f is None:  # complement of the basis span exhausted
                break
            restarts += 1
            space.push_fresh(f)
            continue
        space.extend(w, h_sub)
        if done % stop.check_every == 0 and done < stop.m_a:
            vals, _ = _hessenberg_eigs(H[:done, :done])
            ready, _ = _stop_ready(vals, prev, stop)
            prev = vals
            if ready:
                break
    basis = space.export()
    Hout = H[: done + 1, : done]
    pairs = ritz_pairs(Hout, basis, pol)
    vals = np.array([p[0] for p in pairs])
    converged = (_stop_ready(vals, prev, stop)[1] if prev is not None
                 else int(np.count_nonzero(vals.real >= stop.eps_eig)))
    return ArnoldiResult(H=Hout, basis=basis, rank_trace=ranks, ritz_values=vals,
                         ritz_vectors=[p[1] for p in pairs], converged_count=converged,
                         breakdown=breakdown, iterations=done, diagnostics=diagnostics,
                         restarts=restarts)


def start_vector(n_x: int, n_t: int | None = None, mode: str = "ic", start: str = "ones",
                 seed: int = 0, device=None):
    """Seeded Arnoldi start (cli.py:247-266): all-ones by default, otherwise
    numpy's PCG64 `default_rng(seed).standard_normal`, generated on the host
    (so the bits are the reference's) and normalised.  IC / steady modes give a
    unit n_x vector; source mode a rank-1 field whose two factors have unit
    norm (W1 drawn before W2, as the reference).  `device=None` returns host
    numpy (what the reference returns); a torch device returns device data."""
    if start not in ("ones", "random"):
        raise ValueError(f"start must be 'ones' or 'random', got {start!r}")
    if mode == "source":
        if n_t is None:
            raise ValueError("source mode needs n_t")
        if start == "ones":
            w1 = np.ones((n_x, 1)) / np.sqrt(n_x)
            w2 = np.ones((n_t, 1)) / np.sqrt(n_t)
        else:
            rng = np.random.default_rng(seed)
            w1 = rng.standard_normal((n_x, 1))
            w2 = rng.standard_normal((n_t, 1))
            w1 /= np.linalg.norm(w1)
            w2 /= np.linalg.norm(w2)
        return LowRankMat(w1, w2)
    v = np.ones(n_x) if start == "ones" else np.random.default_rng(seed).standard_normal(n_x)
    v = v / np.linalg.norm(v)
    if device is None:
        return v
    return _torch().as_tensor(v, dtype=_torch().float64).to(device)


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
    tail = np.sqrt(np.cumsum((s ** 2)[::-1]))[::-1]
    r = int(np.count_nonzero(tail > tail_tol * float(np.linalg.norm(s))))
    return r, (float(s[1] / s[0]) if s.size > 1 else 0.0)
