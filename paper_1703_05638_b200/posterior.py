"""Low-rank posterior covariance via Sherman-Morrison-Woodbury (mirrors lrpostcov/posterior.py).

Γ_post v = γ (v - V (λ̃ ∘ Vᵀv)),  diag(Γ_post) = γ (1 - Σ_i λ̃_i V[:, i]²),
λ̃ = λ/(λ+1) (posterior.py:1-9).  Runs once after the Arnoldi recurrence on
the n_x x k Ritz basis; the arithmetic is done with device tensors and the
summary is returned as numpy arrays like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

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

    @property
    def k(self) -> int:
        return self.V.shape[1]


def _torch():
    import torch

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


def variance_diag(eigenvalues, V, gamma_prior: float) -> np.ndarray:
    """γ (1 - Σ λ̃ V²) after re-orthonormalising V (posterior.py:56-62)."""
    torch = _torch()
    Vd = _as_dev(V)
    if Vd.ndim == 1:
        Vd = Vd.reshape(1, -1)
    Vd = _reorthonormalize_dev(Vd)
    filt = np.array([lambda_tilde(float(l)) for l in np.atleast_1d(eigenvalues)])
    if Vd.shape[1] == 0:
        return np.full(Vd.shape[0], gamma_prior)
    f = torch.as_tensor(filt, device=Vd.device)
    return (gamma_prior * (1.0 - (Vd * Vd) @ f)).cpu().numpy()


def build_summary(ritz_values, ritz_vectors, gamma_prior: float, eps_eig: float | None = None,
                  imag_rtol: float = 1e-6, n_x: int | None = None) -> PosteriorSummary:
    """Retain λ >= eps_eig, normalise, re-orthonormalise, variance (posterior.py:65-111)."""
    torch = _torch()
    vals = np.asarray(ritz_values)
    scale = float(np.max(np.abs(vals.real))) if vals.size else 0.0
    if scale > 0 and np.max(np.abs(vals.imag)) > imag_rtol * scale:
        raise NumericalError(
            "Ritz values have a significant imaginary part "
            f"({np.max(np.abs(vals.imag)):.3e} vs scale {scale:.3e})")
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
    if Vd.shape[1]:
        f = torch.as_tensor(filters, device=Vd.device)
        var = (gamma_prior * (1.0 - (Vd * Vd) @ f)).cpu().numpy()
    else:
        var = np.full(Vd.shape[0], gamma_prior)
    return PosteriorSummary(eigenvalues=lams, filters=filters, V=Vd.cpu().numpy(),
                            gamma_prior=gamma_prior, variance_field=var)


def posterior_apply(v, summary: PosteriorSummary) -> np.ndarray:
    """Γ_post v (posterior.py:120-125)."""
    v = np.asarray(v, dtype=float)
    if summary.k == 0:
        return summary.gamma_prior * v
    V = summary.V
    return summary.gamma_prior * (v - V @ (summary.filters * (V.T @ v)))
