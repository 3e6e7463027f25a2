"""TEST INFRASTRUCTURE ONLY -- restatement of ``tensorpde/cp.py`` (CP algebra + ALS).

A CP tensor here is a plain list of factor matrices ``F[k]`` of shape
``(Q_k, r)``; column ``l`` is term ``l`` and scalars live in mode 0
(reference ``cp.py:1-12``).
"""

from __future__ import annotations

import numpy as np

REF_REG = 1e-12  # reference Tikhonov scale, cp.py:166


class ConditioningError(RuntimeError):
    """Mirror of ``cp.ConditioningError`` (cp.py:38-39)."""


def add(f, g):
    """Column concatenation, g's terms after f's (cp.py:98-101)."""
    return [np.hstack([a, b]) for a, b in zip(f, g)]


def scale(f, c):
    """Scalar folded into mode 0 (cp.py:104-108)."""
    out = [fk.copy() for fk in f]
    out[0] = out[0] * c
    return out


def inner_product(f, g):
    """``sum_{l,n} prod_k (F_k^H G_k)[l, n]`` (cp.py:111-121)."""
    acc = None
    for fk, gk in zip(f, g):
        m = fk.conj().T @ gk
        acc = m if acc is None else acc * m
    return complex(acc.sum())


def norm(f):
    """cp.py:124-126."""
    return float(np.sqrt(max(inner_product(f, f).real, 0.0)))


def solve_gram(gram, rhs, lam=None, reg_scale=REF_REG):
    """``(gram + lambda I) X = rhs``.

    ``lam=None`` is the reference rule ``lambda = 1e-12 tr(G)/r``
    (cp.py:169-180, LU via ``np.linalg.solve`` with ``lstsq`` fallback);
    a float is the fixed regulariser the BASELINE configs ask for.
    """
    r = gram.shape[0]
    if lam is None:
        lam = reg_scale * max(np.trace(gram).real, 0.0) / max(r, 1)
    sys = gram + lam * np.eye(r)
    try:
        out = np.linalg.solve(sys, rhs)
    except np.linalg.LinAlgError:
        out = np.linalg.lstsq(sys, rhs, rcond=None)[0]
    if not np.all(np.isfinite(out)):
        raise ConditioningError("normal equations produced non-finite coefficients")
    return out


def als(target, init, sweeps, lam=None, tol=0.0, stall=-np.inf, trace=None):
    """Gauss-Seidel ALS of ``cp_approx_als`` for a CP target (cp.py:266-334).

    ``target`` and ``init`` are factor lists; returns the fitted factor list.
    ``stall=-inf`` and ``tol=0`` run exactly ``sweeps`` sweeps (the BASELINE
    fixed-sweep setting); the defaults of the reference are ``tol=0``,
    ``stall=1e-13``.
    """
    n = len(target)
    r = init[0].shape[1]
    t = [np.asarray(v) for v in target]
    norm_sq = max(inner_product(t, t).real, 0.0)           # _CPTarget.__init__, cp.py:186-188
    t_norm = np.sqrt(norm_sq)
    guess = [u.copy() for u in init]                       # cp.py:301
    grams = [fk.conj().T @ fk for fk in guess]             # cp.py:305
    cross = [gk.conj().T @ tk for gk, tk in zip(guess, t)]  # cp.py:190-191
    prev = np.inf
    for _ in range(sweeps):
        for j in range(n):
            gram = np.ones((r, r), dtype=np.result_type(*guess))
            for k in range(n):
                if k != j:
                    gram = gram * grams[k]                  # cp.py:312-315
            had = np.ones_like(cross[0])
            for k in range(n):
                if k != j:
                    had = had * cross[k]                    # cp.py:197-201
            rhs = had @ t[j].T                              # cp.py:203
            guess[j] = solve_gram(gram, rhs, lam).T         # cp.py:317
            grams[j] = guess[j].conj().T @ guess[j]         # cp.py:318
            cross[j] = guess[j].conj().T @ t[j]             # cp.py:194-195
        self_sq = np.ones((r, r), dtype=grams[0].dtype)
        for g in grams:
            self_sq = self_sq * g
        had = np.ones_like(cross[0])
        for c in cross:
            had = had * c
        ov = complex(had.sum())                             # cp.py:205-209
        resid = float(np.sqrt(max(norm_sq - 2.0 * ov.real + self_sq.sum().real, 0.0)))  # cp.py:325-326
        if trace is not None:
            trace.append(resid)
        if resid <= tol * t_norm:                           # cp.py:329-330
            break
        if prev - resid < stall * max(t_norm, 1.0):         # cp.py:331-332
            break
        prev = resid
    return guess


def random_cp(qs, r, rng, real=False):
    """Normalised random terms (cp.py:129-136); ``real=True`` drops the imaginary draw."""
    out = []
    for q in qs:
        m = rng.standard_normal((q, r))
        if not real:
            m = m + 1j * rng.standard_normal((q, r))
        m = m / np.linalg.norm(m, axis=0, keepdims=True)
        out.append(m)
    return out


def pad_rank(f, r, rng, rel_scale=1e-8, real=False):
    """cp.py:139-146 (``real=True``: real random pad terms)."""
    if r < f[0].shape[1]:
        raise ValueError("cannot pad down")
    if r == f[0].shape[1]:
        return [x.copy() for x in f]
    pad = scale(random_cp([x.shape[0] for x in f], r - f[0].shape[1], rng, real=real),
                rel_scale * max(norm(f), 1.0))
    return add(f, pad)


def relative_error_gram(f, g, nf):
    """Reference Gram-identity error (cp.py:369-375); floor ~1.5e-8, never used as a parity gate."""
    d = inner_product(f, f).real - 2.0 * inner_product(g, f).real + inner_product(g, g).real
    return float(np.sqrt(max(d, 0.0)) / nf)


def rank_reduce(f, r_target, eps, sweeps=200, stall=1e-13, seed=0, real=False):
    """``rank_reduce_als`` (cp.py:337-366): adaptive rank 1..r_target, warm start + one random term."""
    nf = norm(f)
    qs = [x.shape[0] for x in f]
    zero = [np.zeros((q, 1), dtype=f[0].dtype) for q in qs]
    if nf == 0.0:
        return zero
    rng = np.random.default_rng(seed)
    best, best_err = zero, 1.0
    guess = None
    for r in range(1, r_target + 1):
        init = random_cp(qs, 1, rng, real=real) if guess is None else add(guess, random_cp(qs, 1, rng, real=real))
        guess = als(f, init, sweeps, lam=None, tol=0.0, stall=stall)
        err = relative_error_gram(f, guess, nf)
        if err < best_err:
            best, best_err = guess, err
        if err <= eps:
            return guess
    return best
