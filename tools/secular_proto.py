"""Prototype (numpy) of the core SVD by successive column appends solved with
the secular equation (Gu-Eisenstat vectors), checked on real flush cores.

Core of a flush: K = [[diag(S), C], [0, R]] (n = r + p, R upper triangular in
pivot order).  Appending column k of the new block to the SVD of the leading
(r+k) x (r+k) block gives M = [[diag(s), z], [0, rho]], z = U^T c, rho = R[k,k]:
    M M^T = diag(s_0^2, ..., s_{m-1}^2, 0) + w w^T,   w = (z, rho),
so sigma^2 are the roots of f(lam) = 1 + sum_j w_j^2 / (d_j^2 - lam) with
poles d = (s, 0); u_k ~ w_j / (d_j^2 - sigma_k^2), v_k ~ (s_j w_j / (d_j^2 -
sigma_k^2), -1) with w replaced by the Loewner weights recomputed from the
computed roots (numerically orthogonal vectors).
"""
import sys

import numpy as np

EPS = 2.220446049250313e-16


def secular_roots(d, w):
    """Roots of 1 + sum w_j^2/(d_j^2 - lam), d ascending (d_0 may be 0), all
    w_j != 0, distinct d.  Returns (origin index o_i, tau_i) with
    lam_i = d_o^2 + tau_i, plus iteration counts."""
    K = len(d)
    w2 = w * w
    nz2 = float(w2.sum())
    org = np.zeros(K, dtype=int)
    tau = np.zeros(K)
    its = np.zeros(K, dtype=int)
    if K == 1:  # lam = d_0^2 + w_0^2 exactly
        tau[0] = w2[0]
        its[0] = 1
        return org, tau, its
    for i in range(K):
        last = i == K - 1
        if not last:
            gap = (d[i + 1] - d[i]) * (d[i + 1] + d[i])
            # f at the midpoint, differences relative to d_i
            dl = (d - d[i]) * (d + d[i]) - 0.5 * gap
            fm = 1.0 + np.sum(w2 / dl)
            if fm >= 0.0:  # root in (d_i^2, mid): origin d_i, tau in (0, gap/2)
                o, lo, hi = i, 0.0, 0.5 * gap
            else:          # root in (mid, d_{i+1}^2): origin d_{i+1}
                o, lo, hi = i + 1, -0.5 * gap, 0.0
        else:
            o, lo, hi = i, 0.0, nz2
        base = (d - d[o]) * (d + d[o])  # d_j^2 - d_o^2
        # initial guess: the two-pole model around the root with the other
        # poles frozen at the bracket's midpoint, solved exactly
        ia, ib = (i, i + 1) if not last else ((K - 2, K - 1) if K > 1 else (K - 1, K - 1))
        tm = 0.5 * (lo + hi)
        dlm = base - tm
        msk = np.ones(K, bool); msk[ia] = False; msk[ib] = False
        Cc = 1.0 + np.sum(w2[msk] / dlm[msk])
        pa, pb = base[ia], base[ib]          # pole positions relative to the origin
        t = tm
        if ia != ib:
            # Cc + w2a/(pa - t) + w2b/(pb - t) = 0  <=>  Cc (pa-t)(pb-t) + w2a (pb-t) + w2b (pa-t) = 0
            qa = Cc
            qb = -(Cc * (pa + pb) + w2[ia] + w2[ib])
            qc = Cc * pa * pb + w2[ia] * pb + w2[ib] * pa
            cand = []
            if qa != 0.0:
                disc = qb * qb - 4 * qa * qc
                if disc >= 0:
                    sq = np.sqrt(disc)
                    q = -0.5 * (qb + np.copysign(sq, qb))
                    if q != 0.0:
                        cand = [q / qa, qc / q]
            elif qb != 0.0:
                cand = [-qc / qb]
            cand = [c for c in cand if lo < c < hi]
            if cand:
                t = cand[0]
        for it in range(60):
            dl = base - t               # d_j^2 - lam
            terms = w2 / dl
            f = 1.0 + terms.sum()
            dterm = terms / dl          # derivative of each term in lam
            if last:
                psi_m = np.arange(K) < K - 1
            else:
                psi_m = np.arange(K) <= i
            psi, phi = terms[psi_m].sum(), terms[~psi_m].sum()
            dpsi, dphi = dterm[psi_m].sum(), dterm[~psi_m].sum()
            err = 8.0 * (abs(psi) + abs(phi) + 1.0) * EPS * K
            if abs(f) <= err:
                break
            if f > 0:
                hi = min(hi, t)
            else:
                lo = max(lo, t)
            # middle-way rational step on the two poles around the root
            if not last:
                da, db = dl[i], dl[i + 1]
            else:
                da, db = dl[K - 2] if K > 1 else dl[K - 1], dl[K - 1]
            df = dpsi + dphi
            c = f - da * dpsi - db * dphi
            a = (da + db) * f - da * db * df
            b = da * db * f
            disc = np.sqrt(abs(a * a - 4.0 * b * c))
            if not last:
                if c == 0.0:
                    eta = b / a if a != 0.0 else 0.0
                elif a <= 0.0:
                    eta = (a - disc) / (2.0 * c)
                else:
                    eta = 2.0 * b / (a + disc)
            else:
                if c == 0.0:
                    eta = b / a if a != 0.0 else 0.0
                elif a >= 0.0:
                    eta = (a + disc) / (2.0 * c)
                else:
                    eta = 2.0 * b / (a - disc)
            tn = t + eta
            if not (lo < tn < hi) or eta == 0.0 or not np.isfinite(tn):
                tn = 0.5 * (lo + hi)
            if tn == t:
                break
            t = tn
        org[i], tau[i], its[i] = o, t, it + 1
    return org, tau, its


def append_svd(s, z, rho):
    """SVD of M = [[diag(s), z], [0, rho]] -> (sig desc, U, V), M = U diag(sig) V^T."""
    m = len(s)
    N = m + 1
    # pole order: pole j <-> M row/col j (j < m: old, d = s_j); pole m: appended, d = 0
    d = np.concatenate((np.abs(s), [0.0]))
    sgn = np.concatenate((np.sign(s) + (s == 0), [1.0]))  # s_j < 0 handled by a sign flip of v
    w = np.concatenate((z, [rho]))
    tol = 8.0 * EPS * max(d.max(), np.abs(w).max(), 1e-300)
    U = np.eye(N)
    V = np.eye(N)
    if abs(w[m]) < tol:
        w[m] = tol if w[m] >= 0 else -tol
    defl = [(j, j) for j in range(m) if abs(w[j]) <= tol]  # (u column, v column)
    act = [j for j in range(N) if abs(w[j]) > tol or j == m]
    # sort active by d ascending (pole m, d = 0, first)
    act.sort(key=lambda j: (d[j], 0 if j == m else 1))
    # close poles: rotate the pair so the first loses its weight
    k = 1
    zp = m  # the pole whose diagonal column is absent (d = 0): initially the appended one
    while k < len(act):
        a, b = act[k - 1], act[k]
        if d[b] - d[a] <= tol:
            r = np.hypot(w[a], w[b])
            c, sn = w[b] / r, w[a] / r  # new w_a = 0, w_b = r
            G = np.array([[c, -sn], [sn, c]])
            # left rotation of rows (a, b): u-basis; right rotation of cols
            # (a, b) only when both are diagonal columns (a != m)
            U[:, [a, b]] = U[:, [a, b]] @ G.T
            if a != zp:
                V[:, [a, b]] = V[:, [a, b]] @ G.T
                d[a] = d[b]
                defl.append((a, a))
            else:  # zero pole with an old d_b ~ 0: column b becomes zero, b takes the role
                d[b] = 0.0
                defl.append((a, b))
                zp = b
            w[a], w[b] = 0.0, r
            act.pop(k - 1)
        else:
            k += 1
    # deflated: sigma = d_j, u = U e_j, v = V e_j (rows unaffected by w)
    dd = d[act]
    ww = w[act]
    K = len(act)
    org, tau, its = secular_roots(dd, ww)
    lam_minus = np.empty((K, K))  # [i, j] = lam_i - d_j^2
    for i in range(K):
        o = org[i]
        lam_minus[i] = tau[i] - (dd - dd[o]) * (dd + dd[o])
    sig_a = np.sqrt(dd[org] ** 2 + tau)
    # Loewner weights
    zh = np.empty(K)
    for j in range(K):
        prod = lam_minus[K - 1, j]
        for i in range(j):
            prod *= lam_minus[i, j] / ((dd[i] - dd[j]) * (dd[i] + dd[j]))
        for i in range(j, K - 1):
            prod *= lam_minus[i, j] / ((dd[i + 1] - dd[j]) * (dd[i + 1] + dd[j]))
        zh[j] = np.copysign(np.sqrt(max(prod, 0.0)), ww[j])
    Ua = np.zeros((N, K))
    Va = np.zeros((N, K))
    for i in range(K):
        u = zh / (-lam_minus[i])             # w_j / (d_j^2 - lam_i)
        u /= np.linalg.norm(u)
        v = np.zeros(N)
        for jj, j in enumerate(act):
            if j != m:
                v[j] = dd[jj] * zh[jj] / (-lam_minus[i, jj])
        v[m] = -1.0
        v /= np.linalg.norm(v)
        uu = np.zeros(N)
        uu[act] = u
        Ua[:, i] = U @ uu
        Va[:, i] = V @ v
    sig = list(sig_a)
    Ucols = [Ua[:, i] for i in range(K)]
    Vcols = [Va[:, i] for i in range(K)]
    for ju, jv in defl:
        sig.append(0.0 if ju != jv else d[ju])
        Ucols.append(U[:, ju])
        Vcols.append(V[:, jv])
    sig = np.array(sig)
    order = np.argsort(-sig, kind="stable")
    Uo = np.array(Ucols).T[:, order]
    Vo = np.array(Vcols).T[:, order]
    Vo = Vo * sgn[:, None]
    return sig[order], Uo, Vo, its


def core_svd(K, r):
    """SVD of the n x n core [[diag(S), C], [0, R]] by n - r column appends."""
    n = K.shape[0]
    s = np.diag(K)[:r].copy()
    U = np.eye(r)
    V = np.eye(r)
    its_all = []
    for k in range(r, n):
        c = K[:k, k]
        z = U.T @ c
        rho = K[k, k]
        sig, Ut, Vt, its = append_svd(s, z, rho)
        its_all.extend(its)
        Ub = np.zeros((k + 1, k + 1)); Ub[:k, :k] = U; Ub[k, k] = 1.0
        Vb = np.zeros((k + 1, k + 1)); Vb[:k, :k] = V; Vb[k, k] = 1.0
        U = Ub @ Ut
        V = Vb @ Vt
        s = sig
    return s, U, V, its_all


def check(K, r):
    s, U, V, its = core_svd(K, r)
    n = K.shape[0]
    sr = np.linalg.svd(K, compute_uv=False)
    rec = np.linalg.norm(K - (U * s) @ V.T) / np.linalg.norm(K)
    ou = np.abs(U.T @ U - np.eye(n)).max()
    ov = np.abs(V.T @ V - np.eye(n)).max()
    ds = np.abs(s - sr).max() / sr[0]
    return rec, ou, ov, ds, max(its) if its else 0, np.mean(its) if its else 0


if __name__ == "__main__":
    worst = np.zeros(4)
    for tag in ("fwd", "bwd"):
        h = np.fromfile(f"tools/cores/cores.{tag}", dtype=np.float64).reshape(-1, 1 + 32 * 33)
        mits = []
        for f in range(h.shape[0]):
            n = int(h[f, 0])
            if n < 2:
                continue
            K = h[f, 1:].reshape(32, 33)[:n, :n].copy()
            r = n - 4
            # columns of the new block into pivot order: upper triangular R
            R = K[r:, r:]
            perm = np.argsort([np.max(np.nonzero(np.abs(R[:, j]) > 0)[0], initial=-1) for j in range(n - r)], kind="stable")
            Kp = K.copy()
            Kp[:, r:] = K[:, r + perm]
            res = check(Kp, r)
            worst = np.maximum(worst, res[:4])
            mits.append(res[5])
            if f < 3 or res[3] > 1e-14 or res[1] > 1e-13:
                print(tag, f, n, "rec %.1e orthU %.1e orthV %.1e ds %.1e maxit %d meanit %.1f" % res)
        print(tag, "mean iterations per root %.2f" % np.mean(mits))
    print("worst rec %.1e orthU %.1e orthV %.1e ds %.1e" % tuple(worst))
