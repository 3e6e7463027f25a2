"""TEST INFRASTRUCTURE ONLY -- restatement of ``tensorpde/implicit.py`` (fixed-rank implicit ALS step).

Operator pair tables are built from dense real factor matrices (shim S5 of
SURVEY 8(c)): ``pairs[k][e, z] = A_{e,k}^T A_{z,k}`` is the discrete bilinear
pairing that ``pair_matrix`` (basis.py:207-214) computes in closed form for the
Galerkin basis.  ``orientation="reference"`` reproduces ``build_gamma``
verbatim (implicit.py:134-153, which pairs the old iterate with the A-side
index; forcing block implicit.py:140-152); ``orientation="corrected"`` is shim S7 (the normal equations of
``min |A f_new - B f_old|^2``).  Solves are direct ``(M + lam I)`` solves
(shim S6, replacing LSQR at implicit.py:156-164).
"""

from __future__ import annotations

import numpy as np


def build_tables(factors, eta, zeta, qs):
    """implicit.py:94-108 with dense factors: factors[e][k] is None (identity) or (Q,Q)."""
    ra = len(eta)
    pairs, source = [], []
    for k, q in enumerate(qs):
        mats = [np.eye(q) if factors[e][k] is None else factors[e][k] for e in range(ra)]
        tab = np.empty((ra, ra, q, q))
        src = np.empty((ra, q, q))
        for e in range(ra):
            src[e] = mats[e].T            # A_e^T I
            for z in range(ra):
                tab[e, z] = mats[e].T @ mats[z]
        pairs.append(tab)
        source.append(src)
    eta = np.asarray(eta, dtype=float)
    zeta = np.asarray(zeta, dtype=float)
    return dict(pairs=pairs, source=source, KL=np.outer(eta, eta), KR=np.outer(eta, zeta),
                eta=eta, zeta=zeta)


def term_grams(tables, left, right, skip):
    """implicit.py:111-122."""
    ra = tables["KL"].shape[0]
    had = np.ones((ra, ra, left[0].shape[1], right[0].shape[1]))
    for k in range(len(left)):
        if k == skip:
            continue
        had = had * np.einsum("ezsh,sl,hn->ezln", tables["pairs"][k], left[k], right[k], optimize=True)
    return had


def build_M(q, beta_new, tables):
    """implicit.py:125-131 (rank-major, mode-minor blocks)."""
    had = term_grams(tables, beta_new, beta_new, q)
    r = beta_new[q].shape[1]
    qq = beta_new[q].shape[0]
    m = np.einsum("ez,ezji,ezca->iajc", tables["KL"], had, tables["pairs"][q], optimize=True)
    return m.reshape(r * qq, r * qq)


def forcing_block(q, beta_new, tables, forcing, dt):
    """implicit.py:140-152: dt * sum_e eta_e sum_m (prod_{k!=q} beta_k^T S^e_k c_k)[i,m] (S^e_q c_q)[a,m],
    with the source tables S^e_k = pair(E_e, I) (here A_{e,k}^T)."""
    eta = tables["eta"]
    proj = [np.einsum("esh,hm->esm", tables["source"][k], forcing[k], optimize=True) for k in range(len(beta_new))]
    r = beta_new[q].shape[1]
    rows = np.ones((len(eta), r, forcing[0].shape[1]))
    for k in range(len(beta_new)):
        if k == q:
            continue
        rows = rows * np.einsum("si,esm->eim", beta_new[k], proj[k], optimize=True)
    return dt * np.einsum("e,eim,eam->ia", eta, rows, proj[q], optimize=True)


def build_gamma(q, beta_new, beta_old, tables, orientation="corrected", forcing=None, dt=0.0):
    """implicit.py:134-153 (forcing block: forcing_block)."""
    if orientation == "reference":
        had = term_grams(tables, beta_old, beta_new, q)
        gam = np.einsum("ez,ezji,ezca,cj->ia", tables["KR"], had, tables["pairs"][q],
                        beta_old[q], optimize=True)
    elif orientation == "corrected":
        had = term_grams(tables, beta_new, beta_old, q)
        gam = np.einsum("ez,ezij,ezac,cj->ia", tables["KR"], had, tables["pairs"][q],
                        beta_old[q], optimize=True)
    else:
        raise ValueError(orientation)
    if forcing is not None:
        gam = gam + forcing_block(q, beta_new, tables, forcing, dt)
    return gam.reshape(-1)


def converged(beta_int, beta_new):
    """implicit.py:167-177."""
    worst = 0.0
    for a, b in zip(beta_int, beta_new):
        db = float(np.linalg.norm(b - a))
        na = float(np.linalg.norm(a))
        worst = max(worst, (0.0 if db == 0.0 else np.inf) if na == 0.0 else db / na)
    return worst


def step(f_n, tables, sweeps, lam, schedule="gauss-seidel", delta_beta=1.0, eps_tol=0.0,
         orientation="corrected", forcing=None, dt=0.0):
    """implicit.py:222-298 with direct solves; returns (factors, sweeps_done, eps_conv).
    ``forcing``: list of (Q_k, R_f) factors of the source term, scaled by ``dt``."""
    n = len(f_n)
    r = f_n[0].shape[1]
    beta_old = [fk.copy() for fk in f_n]
    beta_new = [fk.copy() for fk in f_n]
    eps_conv = np.inf
    done = 0
    while eps_conv > eps_tol and done < sweeps:
        beta_int = [b.copy() for b in beta_new]
        src = beta_int if schedule == "jacobi" else beta_new
        solved = []
        for q in range(n):
            bn = beta_int if schedule == "jacobi" else beta_new
            m = build_M(q, bn, tables)
            gam = build_gamma(q, bn, beta_old, tables, orientation, forcing, dt)
            x = np.linalg.solve(m + lam * np.eye(m.shape[0]), gam)
            bq = x.reshape(r, -1).T                      # _unvec, implicit.py:218-219
            if schedule == "jacobi":
                solved.append(bq)
            else:
                beta_new[q] = bq
        if schedule == "jacobi":
            for q in range(n):
                beta_new[q] = solved[q]
        del src
        eps_conv = converged(beta_int, beta_new)
        for q in range(n):                               # implicit.py:281-282
            beta_new[q] = beta_int[q] + (beta_new[q] - beta_int[q]) / delta_beta
        done += 1
    return beta_new, done, eps_conv
