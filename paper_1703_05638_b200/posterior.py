"""Low-rank posterior covariance via Sherman-Morrison-Woodbury (mirrors lrpostcov/posterior.py).

Γ_post v = γ (v - V (λ̃ ∘ Vᵀv)),  diag(Γ_post) = γ (1 - Σ_i λ̃_i V[:, i]²),
λ̃ = λ/(λ+1) (posterior.py:1-9).  With the config prior Γ^{1/2} = √γ P,
P = (δI + γ_p L)⁻¹:
Γ_post v = γ P (Pv - V(λ̃ ∘ VᵀPv)),  diag(Γ_post) = γ (diag(P²) - Σ_i λ̃_i (P v_i)²),
with P·X and diag(P²) on the device (lrk_prior_apply / lrk_prior_diag).  Runs once after the Arnoldi recurrence on
the n_x x k Ritz basis; the arithmetic is done with device tensors and the
summary is returned as numpy arrays like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import NumericalError


def lambda_tilde(lam: float) -> float:
    if lam < 0:
        raise NumericalError(
            f"negative eigenvalue {lam} reached the posterior update; "
            "upstream approximation is not positive semidefinite")
    return lam / (lam + 1.0)


@dataclass(frozen=True)
class PosteriorSummary:
    eigenvalues: np.ndarray
    filters: np.ndarray
    V: np.ndarray
    gamma_prior: float
    variance_field: np.ndarray
    prior: object = None  # config prior (hessian.ConfigPrior) or None for γ·I

    @property
    def k(self) -> int:
        return self.V.shape[1]


def _torch():
    import torch

    _lib.require_cuda()
    return torch


def _reorthonormalize_dev(Vd):
    torch = _torch()
    if Vd.shape[1] == 0:
        return Vd
    Q, _ = torch.linalg.qr(Vd)
    return Q


def _as_dev(V):
    torch = _torch()
    t = torch.as_tensor(np.asarray(V) if isinstance(V, np.ndarray) else V, dtype=torch.float64)
    return t.to("cuda")


def _prior_terms(Vd, prior):
    """(P V, diag(P²)) for the config prior, or (V, 1) for the scalar prior."""
    if prior is None:
        return Vd, 1.0
    return prior.apply(Vd, 1), prior.diag(2)


def variance_diag(eigenvalues, V, gamma_prior: float, prior=None) -> np.ndarray:
    """γ (1 - Σ λ̃ V²) after re-orthonormalising V (posterior.py:56-62);
    γ (diag(P²) - Σ λ̃ (P V)²) with the config prior."""
    torch = _torch()
    Vd = _as_dev(V)
    if Vd.ndim == 1:
        Vd = Vd.reshape(1, -1)
    Vd = _reorthonormalize_dev(Vd)
    filt = np.array([lambda_tilde(float(l)) for l in np.atleast_1d(eigenvalues)])
    PV, dP2 = _prior_terms(Vd, prior)
    if Vd.shape[1] == 0:
        base = dP2 if prior is not None else torch.ones(Vd.shape[0], dtype=torch.float64,
                                                         device=Vd.device)
        return (gamma_prior * base).cpu().numpy()
    f = torch.as_tensor(filt, device=Vd.device)
    return (gamma_prior * (dP2 - (PV * PV) @ f)).cpu().numpy()


def build_summary(ritz_values, ritz_vectors, gamma_prior: float, eps_eig: float | None = None,
                  imag_rtol: float = 1e-6, n_x: int | None = None, prior=None) -> PosteriorSummary:
    """Retain λ >= eps_eig, normalise, re-orthonormalise, variance (posterior.py:65-111)."""
    vals = np.asarray(ritz_values)
    scale = float(np.max(np.abs(vals.real))) if vals.size else 0.0
    if scale > 0 and np.max(np.abs(vals.imag)) > imag_rtol * scale:
        raise NumericalError(
            "Ritz values have a significant imaginary part "
            f"({np.max(np.abs(vals.imag)):.3e} vs scale {scale:.3e})")
    torch = _torch()
    real = vals.real.astype(float)
    order = np.argsort(-real)
    threshold = eps_eig if eps_eig is not None else 0.0
    keep = [i for i in order if real[i] >= threshold]
    if keep:
        cols = [_as_dev(ritz_vectors[i]).reshape(-1) for i in keep]
        Vd = torch.stack([c / c.norm() for c in cols], dim=1)
    else:
        if n_x is not None:
            dim = n_x
        elif len(ritz_vectors):
            dim = int(np.asarray(ritz_vectors[0]).shape[0]) if isinstance(ritz_vectors[0], np.ndarray) \
                else int(ritz_vectors[0].shape[0])
        else:
            raise ValueError("cannot infer the spatial dimension from zero vectors")
        Vd = torch.zeros((dim, 0), dtype=torch.float64, device="cuda")
    Vd = _reorthonormalize_dev(Vd)
    lams = real[keep]
    filters = np.array([lambda_tilde(float(l)) for l in lams])
    PV, dP2 = _prior_terms(Vd, prior)
    if Vd.shape[1]:
        f = torch.as_tensor(filters, device=Vd.device)
        var = (gamma_prior * (dP2 - (PV * PV) @ f)).cpu().numpy()
    elif prior is not None:
        var = (gamma_prior * dP2).cpu().numpy()
    else:
        var = np.full(Vd.shape[0], gamma_prior)
    return PosteriorSummary(eigenvalues=lams, filters=filters, V=Vd.cpu().numpy(),
                            gamma_prior=gamma_prior, variance_field=var, prior=prior)


def posterior_apply(v, summary: PosteriorSummary) -> np.ndarray:
    """Γ_post v (posterior.py:120-125); γ P (Pv - V(λ̃ ∘ VᵀPv)) with the config prior."""
    v = np.asarray(v, dtype=float)
    P = summary.prior
    if P is not None:
        torch = _torch()
        pv = P.apply(_as_dev(v).reshape(-1, 1), 1)
        if summary.k:
            V = _as_dev(summary.V)
            f = torch.as_tensor(summary.filters, device=V.device)
            pv = pv - V @ (f[:, None] * (V.T @ pv))
        return (summary.gamma_prior * P.apply(pv, 1)).reshape(-1).cpu().numpy()
    if summary.k == 0:
        return summary.gamma_prior * v
    V = summary.V
    return summary.gamma_prior * (v - V @ (summary.filters * (V.T @ v)))


# ------------------------------------------------------------------- writers
def variance_to_grid(field_values, n_side: int) -> np.ndarray:
    """Dof-ordered field -> (x2, x1)-indexed n_side x n_side grid (posterior.py:128-130)."""
    return np.asarray(field_values, dtype=float).reshape(n_side, n_side)


def write_variance_csv(field_values, n_side: int, path) -> None:
    """Header c0..c{n-1}, then row j = x2 level j with 17 significant digits (posterior.py:133-139)."""
    lines = [",".join(f"c{i}" for i in range(n_side))]
    lines += [",".join(f"{v:.17g}" for v in row) for row in variance_to_grid(field_values, n_side)]
    with open(path, "w") as fh:
        fh.write("".join(line + "\n" for line in lines))


def write_variance_pgm(field_values, n_side: int, gamma_prior: float, path) -> None:
    """Plain-text 8-bit PGM: the field minimum maps to 0, gamma_prior to 255; a field with no
    reduction anywhere is all white (posterior.py:142-155)."""
    g = variance_to_grid(field_values, n_side)
    lo = float(g.min())
    span = gamma_prior - lo
    pix = np.full(g.shape, 255.0) if span <= 0 else np.clip(255.0 * (g - lo) / span, 0.0, 255.0)
    rows = [" ".join(str(int(v)) for v in row) for row in np.rint(pix)]
    with open(path, "w") as fh:
        fh.write(f"P2\n{n_side} {n_side}\n255\n" + "".join(r + "\n" for r in rows))
