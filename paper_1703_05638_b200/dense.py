"""Dense brute-force cross-check on the GPU for small instances.

Counterpart of lrpostcov/oracle.py:22-320 (dense_misfit_ic / _source /
_steady, dense_eig_top, dense_posterior_diag, compare, hv_agreement), same
names, arguments and report text, so `cli oracle` writes the reference's
oracle_report.txt.  It shares no code with the low-rank device path: the
misfit Hessian is built column-block-wise from the ASSEMBLED spatial matrix
with one dense LU (torch.linalg on the device; all n columns march through
the time loop together as one n x n right-hand side), and everything after it
is plain dense linear algebra.  Dimension cap as the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidConfigError, NumericalError

DENSE_DIM_CAP = 2000


def _torch():
    import torch

    from . import _lib

    _lib.require_cuda()
    return torch


def _guard(dim: int) -> None:
    if dim > DENSE_DIM_CAP:
        raise InvalidConfigError(f"dense oracle dimension {dim} exceeds the cap {DENSE_DIM_CAP}")


def _dev(x):
    torch = _torch()
    return torch.as_tensor(np.asarray(x, dtype=float), dtype=torch.float64, device="cuda")


class _StepLU:
    """One dense LU of the step matrix A = m (I + tau L); solves with A or A^T."""

    def __init__(self, L_dense, m_scale: float, tau: float):
        torch = _torch()
        L = _dev(L_dense)
        n = L.shape[0]
        A = m_scale * (torch.eye(n, dtype=torch.float64, device="cuda") + tau * L)
        self.n, self.m = n, m_scale
        self._lu = torch.linalg.lu_factor(A)
        self._lut = torch.linalg.lu_factor(A.T.contiguous())

    def solve(self, B, transpose: bool = False):
        torch = _torch()
        lu, piv = self._lut if transpose else self._lu
        return torch.linalg.lu_solve(lu, piv, B)


def _march(step: _StepLU, F_of_k, n_t: int, adjoint: bool):
    """Block substitution y_k = A^{-1}(m y_{k±1} + F_k) for a block of right-hand
    sides at once; returns the list of panes indexed by time step."""
    torch = _torch()
    prev = None
    out = [None] * n_t
    order = range(n_t - 1, -1, -1) if adjoint else range(n_t)
    for k in order:
        rhs = F_of_k(k)
        if prev is not None:
            rhs = step.m * prev if rhs is None else step.m * prev + rhs
        if rhs is None:
            rhs = torch.zeros((step.n, step.n), dtype=torch.float64, device="cuda")
        prev = step.solve(rhs, transpose=adjoint)
        out[k] = prev
    return out


def dense_forward(L_dense, m_scale: float, tau: float, F, adjoint: bool = False) -> np.ndarray:
    """Y with K vec(Y) = vec(F) (K^T when adjoint) by block substitution with one dense LU
    of the step matrix (oracle.py:22-39); F and Y are n_x x n_t, one column per time step."""
    Fd = _dev(F)
    n_x, n_t = Fd.shape
    _guard(n_x)
    step = _StepLU(L_dense, m_scale, tau)
    panes = _march(step, lambda k: Fd[:, k:k + 1], n_t, adjoint)
    return _torch().cat(panes, dim=1).cpu().numpy()


def _sym(H):
    """(symmetrised matrix as numpy, asymmetry defect relative to max |H|)."""
    scale = float(H.abs().max())
    defect = float((H - H.T).abs().max() / scale) if scale > 0 else 0.0
    return (0.5 * (H + H.T)).cpu().numpy(), defect


def dense_misfit_ic(L_dense, m_scale: float, tau: float, n_t: int, mask, beta_noise: float,
                    gamma_prior: float):
    """Explicit prior-preconditioned misfit Hessian, IC parameter (oracle.py:60-79):
    all n_x unit vectors go through forward sweep, observation weight and
    adjoint sweep together."""
    torch = _torch()
    n_x = np.asarray(L_dense).shape[0]
    _guard(n_x)
    step = _StepLU(L_dense, m_scale, tau)
    sg = float(np.sqrt(gamma_prior))
    eye = torch.eye(n_x, dtype=torch.float64, device="cuda")
    # forward: the first block's right-hand side is m * sqrt(g) * I
    Y = _march(step, lambda k: (m_scale * sg) * eye if k == 0 else None, n_t, adjoint=False)
    w = beta_noise * tau * m_scale
    mk = _dev(np.asarray(mask, dtype=float))[:, None]
    Q = _march(step, lambda k: w * (mk * Y[k]), n_t, adjoint=True)
    return _sym(sg * m_scale * Q[0])


def dense_misfit_source(L_dense, m_scale: float, tau: float, n_t: int, mask, beta_noise: float,
                        gamma_prior: float):
    """Explicit misfit Hessian for the space-time source parameter (oracle.py:82-109);
    unknowns ordered time-major over space (column-major vec of the n_x x n_t field)."""
    torch = _torch()
    n_x = np.asarray(L_dense).shape[0]
    dim = n_x * n_t
    _guard(dim)
    step = _StepLU(L_dense, m_scale, tau)
    inj = float(np.sqrt(gamma_prior)) * tau * m_scale
    w = beta_noise * tau * m_scale
    mk = _dev(np.asarray(mask, dtype=float))[:, None]
    eye = torch.eye(n_x, dtype=torch.float64, device="cuda")
    H = torch.zeros((dim, dim), dtype=torch.float64, device="cuda")
    for j in range(n_t):  # the n_x unit sources placed at time step j
        Y = _march(step, lambda k: inj * eye if k == j else None, n_t, adjoint=False)
        Q = _march(step, lambda k: w * (mk * Y[k]), n_t, adjoint=True)
        for k in range(n_t):
            H[k * n_x:(k + 1) * n_x, j * n_x:(j + 1) * n_x] = inj * Q[k]
    return _sym(H)


def dense_misfit_steady(L_dense, beta_noise: float, beta_prior: float):
    """(beta_prior / beta_noise) L^{-1} L^{-1} (oracle.py:112-118)."""
    torch = _torch()
    L = _dev(L_dense)
    _guard(L.shape[0])
    Li = torch.linalg.inv(L)
    return _sym((beta_prior / beta_noise) * (Li @ Li))


def dense_eig_top(Hd, k: int):
    """Top-k eigenpairs of a symmetric matrix, descending, residual-checked (oracle.py:134-152)."""
    torch = _torch()
    Hn = np.asarray(Hd, dtype=float)
    if not np.allclose(Hn, Hn.T, atol=1e-10 * max(1.0, np.abs(Hn).max())):
        raise InvalidConfigError("dense_eig_top expects a symmetric matrix")
    H = _dev(Hn)
    try:
        vals, vecs = torch.linalg.eigh(H)
    except RuntimeError as exc:
        raise NumericalError(f"dense symmetric eigensolve failed: {exc}") from exc
    vals, vecs = vals.flip(0), vecs.flip(1)
    k = min(k, vals.numel())
    norm = max(float(vals.abs().max()), 1e-300)
    res = (H @ vecs[:, :k] - vecs[:, :k] * vals[:k]).norm(dim=0)
    bad = (res > 1e-10 * norm).nonzero()
    if bad.numel():
        i = int(bad[0])
        raise NumericalError(f"dense eigenpair {i} residual {float(res[i]):.3e} above tolerance")
    return vals[:k].cpu().numpy(), vecs[:, :k].cpu().numpy()


def dense_posterior_diag(H_preconditioned, gamma_prior: float) -> np.ndarray:
    """diag (H/gamma + I/gamma)^{-1} (oracle.py:155-160)."""
    torch = _torch()
    H = _dev(H_preconditioned)
    n = H.shape[0]
    post = torch.linalg.inv(H / gamma_prior + torch.eye(n, dtype=torch.float64, device="cuda") / gamma_prior)
    return post.diagonal().cpu().numpy().copy()


@dataclass
class OracleReport:
    """Error metrics of the low-rank path against the dense path (oracle.py:176-204)."""

    eig_rel_errors: np.ndarray
    max_eig_rel_error: float
    max_principal_angle: float
    max_pair_residual: float
    variance_rel_error: float | None
    hv_rel_error: float | None
    tolerances: dict = field(default_factory=dict)
    passed: bool = False

    def as_text(self) -> str:
        rows = [("max_eig_rel_error", self.max_eig_rel_error),
                ("max_principal_angle", self.max_principal_angle),
                ("max_pair_residual", self.max_pair_residual)]
        if self.variance_rel_error is not None:
            rows.append(("variance_rel_error", self.variance_rel_error))
        if self.hv_rel_error is not None:
            rows.append(("hv_rel_error", self.hv_rel_error))
        rows += [(f"tol_{k}", v) for k, v in self.tolerances.items()]
        text = "".join(f"{k}={v:.6e}\n" for k, v in rows)
        return text + f"result={'PASS' if self.passed else 'FAIL'}\n"


def _degenerate_groups(vals, rel_gap: float):
    """Index ranges of near-equal consecutive values of a descending spectrum."""
    cuts = [0]
    for i in range(1, len(vals)):
        big = max(abs(vals[i - 1]), abs(vals[i]), 1e-300)
        if abs(vals[i - 1] - vals[i]) > rel_gap * big:
            cuts.append(i)
    cuts.append(len(vals))
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def _largest_principal_angle(A, B) -> float:
    """Largest principal angle between span(A) and span(B) (sine-based, accurate
    for small angles): asin of the largest singular value of (I - Qa Qa^T) Qb."""
    torch = _torch()
    Qa, _ = torch.linalg.qr(_dev(A))
    Qb, _ = torch.linalg.qr(_dev(B))
    R = Qb - Qa @ (Qa.T @ Qb)
    s = torch.linalg.svdvals(R)
    return float(torch.asin(s.max().clamp(max=1.0))) if s.numel() else 0.0


def compare(lr_values, lr_vectors, dense_values, dense_vectors, Hd=None, lr_variance=None,
            dense_variance=None, hv_rel_error=None, eig_rtol: float = 1e-6,
            angle_tol: float = 1e-4, var_rtol: float = 1e-4, hv_rtol: float = 1e-8,
            cluster_gap: float = 1e-3) -> OracleReport:
    """Top-k comparison, k = len(dense_values) (oracle.py:207-288): eigenvalues index
    by index, eigenvector spans per near-degenerate cluster."""
    k = len(dense_values)
    lr_vals = np.asarray(lr_values, dtype=float)[:k]
    lr_vectors = np.asarray(lr_vectors)
    if lr_vals.shape[0] != k or lr_vectors.shape[1] < k:
        raise ValueError(f"low-rank side provides {lr_vals.shape[0]} values / "
                         f"{lr_vectors.shape[1]} vectors, dense side expects {k}")
    dn = np.asarray(dense_values, dtype=float)
    eig_err = np.abs(lr_vals - dn) / np.maximum(np.abs(dn), 1e-300)
    angle = 0.0
    for a, b in _degenerate_groups(dn, cluster_gap):
        if b <= lr_vectors.shape[1]:
            angle = max(angle, _largest_principal_angle(lr_vectors[:, a:b], dense_vectors[:, a:b]))
    resid = 0.0
    if Hd is not None and k:
        V = lr_vectors[:, :k]
        R = np.asarray(Hd) @ V - V * lr_vals
        resid = float(np.linalg.norm(R, axis=0).max() / max(abs(dn[0]), 1e-300))
    var_err = None
    if lr_variance is not None and dense_variance is not None:
        var_err = float(np.max(np.abs(lr_variance - dense_variance) / np.abs(dense_variance)))
    tol = {"eig_rel": eig_rtol, "angle": angle_tol}
    ok = bool(np.all(eig_err <= eig_rtol)) and angle <= angle_tol
    if var_err is not None:
        tol["var_rel"] = var_rtol
        ok = ok and var_err <= var_rtol
    if hv_rel_error is not None:
        tol["hv_rel"] = hv_rtol
        ok = ok and hv_rel_error <= hv_rtol
    return OracleReport(eig_rel_errors=eig_err,
                        max_eig_rel_error=float(eig_err.max()) if eig_err.size else 0.0,
                        max_principal_angle=angle, max_pair_residual=resid,
                        variance_rel_error=var_err, hv_rel_error=hv_rel_error,
                        tolerances=tol, passed=ok)


def hv_agreement(apply, Hd, n_probe: int = 20, seed: int = 0) -> float:
    """Largest relative disagreement of the matrix-free apply with the dense
    matrix over seeded unit probes (oracle.py:291-310) — gate before any
    eigen comparison."""
    rng = np.random.default_rng(seed)
    Hn = np.asarray(Hd)
    worst = 0.0
    for _ in range(n_probe):
        v = rng.standard_normal(Hn.shape[0])
        v /= np.linalg.norm(v)
        ref = Hn @ v
        got = np.asarray(apply(v))
        worst = max(worst, float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)))
    return worst
