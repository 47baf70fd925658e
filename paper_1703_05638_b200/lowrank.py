"""Low-rank factor algebra on the device (mirrors lrpostcov/lowrank.py).

A field Y = W1 W2ᵀ is stored as two fp64 CUDA tensors in column-major layout
(every spatial column contiguous, which is what the kernels stream).  The
public names, signatures and semantics follow the reference:
TruncationPolicy (lowrank.py:25-36), LowRankMat (:39-78), lr_truncate
(:124-144, with _rank_cut :98-111 and _svd_flip :114-121), lr_add (:147-154),
lr_scale (:157-160), lr_dot (:163-168), lr_norm (:171-173),
lr_singular_values (:176-182).  Truncation and inner products run in
liblrk.so; concatenation/scaling are plain device tensor copies.
"""

from __future__ import annotations

from ctypes import byref, c_double, c_int
from dataclasses import dataclass

import numpy as np

from . import _lib

NOISE_FLOOR = 1e-15
CORE_MAX = 160  # widest concatenation the device truncation accepts


def _torch():
    import torch

    return torch


def colmajor(n: int, cap: int, device=None):
    """Uninitialised (n, cap) fp64 CUDA tensor with unit row stride."""
    torch = _torch()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.empty((max(cap, 0), n), dtype=torch.float64, device=dev).T


def to_device_colmajor(X):
    """numpy / torch (n, r) -> fp64 CUDA column-major tensor (copy if needed)."""
    torch = _torch()
    _lib.require_cuda()
    t = torch.as_tensor(X, dtype=torch.float64)
    if t.ndim == 1:
        t = t.reshape(1, -1)  # np.atleast_2d semantics of the reference
    if t.device.type != "cuda":
        t = t.to("cuda")
    if t.ndim != 2:
        raise ValueError(f"factor must be 2-D, got shape {tuple(t.shape)}")
    if t.stride(0) != 1 or (t.shape[1] > 1 and t.stride(1) < max(t.shape[0], 1)):
        t = t.T.contiguous().T
    return t


def _shape_of(X):
    """Anything with .shape as is; nested lists through numpy (host-side shape checks)."""
    return X if hasattr(X, "shape") else np.asarray(X)


def ld_of(t) -> int:
    """Leading dimension (column stride) of a column-major tensor."""
    if t.shape[1] <= 1:
        return max(int(t.shape[0]), 1)
    return int(t.stride(1))


@dataclass(frozen=True)
class TruncationPolicy:
    """Relative Frobenius tolerance eps0 plus an optional hard rank cap."""

    eps0: float = 1e-8
    r_max: int | None = None

    def __post_init__(self):
        if not (0.0 < self.eps0 < 1.0):
            raise ValueError(f"eps0 must lie in (0, 1), got {self.eps0}")
        if self.r_max is not None and self.r_max < 0:
            raise ValueError(f"r_max must be nonnegative, got {self.r_max}")

    @property
    def r_max_c(self) -> int:
        return -1 if self.r_max is None else int(self.r_max)


class LowRankMat:
    """Immutable-by-convention factor pair representing W1 @ W2.T on the device."""

    __slots__ = ("W1", "W2")

    def __init__(self, W1, W2):
        # shape errors are host logic (lowrank.py:47-50): report them before touching the device
        s1, s2 = tuple(_shape_of(W1).shape), tuple(_shape_of(W2).shape)
        if len(s1) > 2 or len(s2) > 2 or (s1[-1] if s1 else 1) != (s2[-1] if s2 else 1):
            raise ValueError(f"factor shapes {s1} and {s2} are inconsistent")
        W1 = to_device_colmajor(W1)
        W2 = to_device_colmajor(W2)
        if W1.shape[1] != W2.shape[1]:
            raise ValueError(
                f"factor shapes {tuple(W1.shape)} and {tuple(W2.shape)} are inconsistent"
            )
        self.W1 = W1
        self.W2 = W2

    @classmethod
    def _wrap(cls, W1, W2) -> "LowRankMat":
        obj = cls.__new__(cls)
        obj.W1 = W1
        obj.W2 = W2
        return obj

    @property
    def r(self) -> int:
        return int(self.W1.shape[1])

    @property
    def shape(self) -> tuple[int, int]:
        return (int(self.W1.shape[0]), int(self.W2.shape[0]))

    @classmethod
    def zeros(cls, n_x: int, n_t: int) -> "LowRankMat":
        return cls._wrap(colmajor(n_x, 0), colmajor(n_t, 0))

    @classmethod
    def from_column(cls, col, n_t: int, k: int) -> "LowRankMat":
        torch = _torch()
        c = to_device_colmajor(torch.as_tensor(col, dtype=torch.float64).reshape(-1, 1))
        e = colmajor(n_t, 1)
        e.zero_()
        e[k, 0] = 1.0
        return cls._wrap(c, e)

    def column(self, k: int):
        """Dense spatial column at time index k (device tensor)."""
        return self.W1 @ self.W2[k, :]

    def dense(self):
        return self.W1 @ self.W2.T

    def numpy(self):
        return self.W1.cpu().numpy(), self.W2.cpu().numpy()

    def _c(self) -> _lib.lrk_lr:
        d = _lib.lrk_lr()
        d.W1 = self.W1.data_ptr() if self.r else None
        d.W2 = self.W2.data_ptr() if self.r else None
        d.ld1 = ld_of(self.W1)
        d.ld2 = ld_of(self.W2)
        d.n_x, d.n_t = self.shape
        d.r = self.r
        d.cap = self.r
        return d

    def __repr__(self) -> str:
        return f"LowRankMat(shape={self.shape}, r={self.r})"


def _out_pair(n_x: int, n_t: int, cap: int):
    W1 = colmajor(n_x, cap)
    W2 = colmajor(n_t, cap)
    d = _lib.lrk_lr()
    d.W1 = W1.data_ptr() if cap else None
    d.W2 = W2.data_ptr() if cap else None
    d.ld1 = max(n_x, 1)
    d.ld2 = max(n_t, 1)
    d.n_x, d.n_t, d.r, d.cap = n_x, n_t, 0, cap
    return W1, W2, d


def _check_same_shape(A: LowRankMat, B: LowRankMat) -> None:
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch: {A.shape} vs {B.shape}")


def lr_to_dense(A: LowRankMat) -> np.ndarray:
    if A.r == 0:
        return np.zeros(A.shape)
    return A.dense().cpu().numpy()


def lr_truncate(A: LowRankMat, pol: TruncationPolicy, flags: int = 0) -> LowRankMat:
    """Recompress to canonical form: ||A - out||_F <= eps0 ||A||_F (lowrank.py:124-144).

    Inputs wider than the 160-column device core go through the fused
    concatenate-and-truncate entry point, which reduces the width exactly
    (dense product on a short side, or rounding-floor folds) before the one
    policy truncation — the reference truncates the whole input once.
    """
    n_x, n_t = A.shape
    if A.r == 0:
        return LowRankMat.zeros(n_x, n_t)
    if A.r > CORE_MAX:
        return lr_add_truncate([A], None, pol)
    ctx = _lib.algebra_context()
    cap = A.r if pol.r_max is None else max(min(A.r, pol.r_max), 1)
    W1, W2, out = _out_pair(n_x, n_t, cap)
    r = c_int(0)
    _lib.check(
        _lib.get_lib().lrk_truncate(ctx.handle, byref(A._c()), byref(out), float(pol.eps0),
                                    pol.r_max_c, int(flags), byref(r), _lib.stream_handle()),
        ctx.handle, "lr_truncate",
    )
    return LowRankMat._wrap(W1[:, : r.value], W2[:, : r.value])


def lr_add_truncate(terms, coefs, pol: TruncationPolicy) -> LowRankMat:
    """truncate(sum_i coefs[i] * terms[i]) with ONE truncation of the whole
    concatenation (lr_add chains + lr_truncate, lowrank.py:147-154/:124-144),
    fused on the device (lrk_add_truncate); coefs None = all ones."""
    terms = list(terms)
    if not terms:
        raise ValueError("lr_add_truncate needs at least one term")
    n_x, n_t = terms[0].shape
    for t in terms[1:]:
        _check_same_shape(terms[0], t)
    R = sum(t.r for t in terms)
    if R == 0:
        return LowRankMat.zeros(n_x, n_t)
    ctx = _lib.algebra_context()
    cap = min(R, CORE_MAX, n_x, n_t)
    if pol.r_max is not None:
        cap = max(min(cap, pol.r_max), 1)
    W1, W2, out = _out_pair(n_x, n_t, max(cap, 1))
    arr = (_lib.lrk_lr * len(terms))(*[t._c() for t in terms])
    cf = None if coefs is None else (c_double * len(terms))(*[float(c) for c in coefs])
    r = c_int(0)
    _lib.check(
        _lib.get_lib().lrk_add_truncate(ctx.handle, len(terms), arr, cf, float(pol.eps0),
                                        pol.r_max_c, byref(out), byref(r), _lib.stream_handle()),
        ctx.handle, "lr_add_truncate",
    )
    return LowRankMat._wrap(W1[:, : r.value], W2[:, : r.value])


def lr_from_dense(X, pol: TruncationPolicy) -> LowRankMat:
    """Compress a dense matrix under the policy (lowrank.py:90-95): the field
    (X, I) with the identity on the shorter side (skips that side's QR)."""
    torch = _torch()
    Xd = to_device_colmajor(X)
    n_x, n_t = Xd.shape
    if n_t <= CORE_MAX or n_t <= n_x:
        eye = to_device_colmajor(torch.eye(n_t, dtype=torch.float64))
        return lr_truncate(LowRankMat._wrap(Xd, eye), pol, flags=_lib.LRK_TRUNC_W2_ORTHOSCALED)
    eye = to_device_colmajor(torch.eye(n_x, dtype=torch.float64))
    return lr_truncate(LowRankMat._wrap(eye, to_device_colmajor(Xd.T)), pol,
                       flags=_lib.LRK_TRUNC_W1_ORTHO)


def lr_add(A: LowRankMat, B: LowRankMat) -> LowRankMat:
    """Exact sum by factor concatenation (lowrank.py:147-154)."""
    _check_same_shape(A, B)
    if A.r == 0:
        return B
    if B.r == 0:
        return A
    n_x, n_t = A.shape
    W1 = colmajor(n_x, A.r + B.r)
    W2 = colmajor(n_t, A.r + B.r)
    W1[:, : A.r] = A.W1
    W1[:, A.r:] = B.W1
    W2[:, : A.r] = A.W2
    W2[:, A.r:] = B.W2
    return LowRankMat._wrap(W1, W2)


def lr_scale(A: LowRankMat, c: float) -> LowRankMat:
    if c == 0.0:
        return LowRankMat.zeros(*A.shape)
    return LowRankMat._wrap(A.W1, A.W2 * float(c))


def lr_dot(A: LowRankMat, B: LowRankMat) -> float:
    """<vec(A), vec(B)> = sum((A1ᵀB1) ∘ (A2ᵀB2)), computed on the device."""
    _check_same_shape(A, B)
    if A.r == 0 or B.r == 0:
        return 0.0
    ctx = _lib.algebra_context()
    out = c_double(0.0)
    _lib.check(
        _lib.get_lib().lrk_dot(ctx.handle, byref(A._c()), byref(B._c()), byref(out),
                               _lib.stream_handle()),
        ctx.handle, "lr_dot",
    )
    return float(out.value)


def lr_norm(A: LowRankMat) -> float:
    return float(np.sqrt(max(lr_dot(A, A), 0.0)))


def lr_singular_values(A: LowRankMat) -> np.ndarray:
    if A.r == 0:
        return np.zeros(0)
    if A.r > CORE_MAX:
        raise NotImplementedError("lr_singular_values supports rank <= 160 on the device")
    ctx = _lib.algebra_context()
    buf = (c_double * A.r)()
    n = c_int(0)
    _lib.check(
        _lib.get_lib().lrk_singular_values(ctx.handle, byref(A._c()), buf, A.r, byref(n),
                                           _lib.stream_handle()),
        ctx.handle, "lr_singular_values",
    )
    return np.array(buf[: n.value])
