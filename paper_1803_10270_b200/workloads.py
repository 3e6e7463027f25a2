"""Seeded synthetic inputs for the five BASELINE configs (BASELINE.json:configs).

Everything is generated on the host with ``numpy.random.default_rng(seed)`` so
the GPU path and the CPU oracle consume identical bytes.  The
functions return plain numpy arrays; callers upload them.
"""

from __future__ import annotations

import numpy as np

from .basis import BasisSpec, fourier_diff_matrix, nodes


def cfg1(seed: int = 0, d: int = 6, Q: int = 256, R: int = 512, r: int = 32):
    """Standalone CP-ALS truncation: V_k ~ N(0,1)/sqrt(Q), init = first r terms."""
    rng = np.random.default_rng(seed)
    V = [rng.standard_normal((Q, R)) / np.sqrt(Q) for _ in range(d)]
    init = [v[:, :r].copy() for v in V]
    specs = tuple(BasisSpec(Q, np.pi, "collocation", lo=0.0) for _ in range(d))
    return dict(specs=specs, V=V, init=init, r=r, sweeps=20, lam=1e-10)


ADV_A = (1.0, 0.5, -0.75, 0.25, -1.0, 0.8)


def advection_ic(seed: int, Q: int, d: int = 6, rank: int = 3, r: int = 6):
    """Rank-3 IC w_k prod_j exp(sin(x_j + phi_kj)), padded to rank r with
    1e-8-scaled real N(0,1) terms (BASELINE cfg0/cfg2)."""
    rng = np.random.default_rng(seed)
    x = 2 * np.pi * np.arange(Q) / Q
    w = rng.uniform(0.5, 1.5, size=rank)
    phi = rng.uniform(0, 2 * np.pi, size=(rank, d))
    factors = []
    for j in range(d):
        cols = np.stack([np.exp(np.sin(x + phi[kk, j])) for kk in range(rank)], axis=1)
        if j == 0:
            cols = cols * w
        factors.append(cols)
    pad = [1e-8 * rng.standard_normal((Q, r - rank)) for _ in range(d)]
    factors = [np.hstack([f, p]) for f, p in zip(factors, pad)]
    return dict(factors=factors, w=w, phi=phi, x=x)


def advection_exact(ic, t: float, a=ADV_A):
    """Exact solution u(x, t) = u0(x - a t): phases shifted by -a_j t (rank-3 CP)."""
    rank = len(ic["w"])
    d = ic["phi"].shape[1]
    x = ic["x"]
    out = []
    for j in range(d):
        cols = np.stack([np.exp(np.sin(x - a[j] * t + ic["phi"][kk, j])) for kk in range(rank)], axis=1)
        if j == 0:
            cols = cols * ic["w"]
        out.append(cols)
    return out


def cfg0(seed: int = 0):
    Q, d = 32, 6
    specs = tuple(BasisSpec(Q, np.pi, "collocation", lo=0.0) for _ in range(d))
    ic = advection_ic(seed, Q, d, 3, 6)
    return dict(specs=specs, ic=ic, a=ADV_A, D=fourier_diff_matrix(Q), dt=1e-3, steps=100, r=6,
                sweeps=10, lam=1e-10)


def cfg2(seed: int = 0):
    Q, d = 128, 6
    specs = tuple(BasisSpec(Q, np.pi, "collocation", lo=0.0) for _ in range(d))
    ic = advection_ic(seed, Q, d, 3, 16)
    return dict(specs=specs, ic=ic, a=ADV_A, D=fourier_diff_matrix(Q), dt=1e-2, steps=50, r=16,
                sweeps=20, lam=1e-10)


def maxwellian_1d(v):
    return np.exp(-0.5 * v * v) / np.sqrt(2.0 * np.pi)


def bgk_operator_terms(Qx: int = 64, Qv: int = 64, vmax: float = 6.0, nu: float = 1.0):
    """Separable terms of L = -sum_i diag(v_i)(x) D_{x_i}  - nu I + nu P  (BASELINE cfg3).

    Modes are (x1, x2, x3, v1, v2, v3); x on the periodic grid 2 pi j / Qx with the
    Fourier collocation derivative, v on linspace(-vmax, vmax, Qv) with trapezoid
    weights.  P projects (in v, identity in x) onto M(v) span{1, v1, v2, v3, psi},
    psi = |v|^2 - c, orthogonal under the DISCRETE measure w M so that P is an
    exact projection on the grid: P = sum_m (M phi_m)(w phi_m)^T / g_m, which
    separates into 1 + 3 + 16 rank-1-per-mode terms.  Returns (weights, mats)
    with mats[t][k] a dense (Q, Q) matrix or None (identity).
    """
    D = fourier_diff_matrix(Qx)
    v = np.linspace(-vmax, vmax, Qv)
    w = np.full(Qv, v[1] - v[0])
    w[0] *= 0.5
    w[-1] *= 0.5
    M1 = maxwellian_1d(v)
    wm = w * M1
    m0, m2 = wm.sum(), (wm * v * v).sum()
    mass3 = m0 ** 3
    # psi = sum_i v_i^2 - c with c making <1, psi> = 0 under the product measure
    c = 3.0 * m2 / m0
    ones = np.ones(Qv)
    weights, mats = [], []
    # transport: -v_i d/dx_i
    for i in range(3):
        row = [None] * 6
        row[i] = D
        row[3 + i] = np.diag(v)
        weights.append(-1.0)
        mats.append(row)
    # relaxation: -nu I
    weights.append(-nu)
    mats.append([None] * 6)

    def outer(a, b):                       # (M a)(w b)^T on one velocity mode
        return np.outer(M1 * a, w * b)

    # P terms: phi_0 = 1 (norm g0 = m0^3)
    weights.append(nu / mass3)
    mats.append([None, None, None, outer(ones, ones), outer(ones, ones), outer(ones, ones)])
    # phi_i = v_i (norm g = m2 m0^2)
    for i in range(3):
        row = [None, None, None] + [outer(ones, ones)] * 3
        row[3 + i] = outer(v, v)
        weights.append(nu / (m2 * m0 * m0))
        mats.append(row)
    # psi = sum_i v_i^2 - c: norm g4 = <psi, psi>
    pieces = [v * v, ones]
    # <psi,psi> = sum_{i,j} <v_i^2 v_j^2> - 2c sum_i <v_i^2> + c^2 <1>
    m4 = (wm * v ** 4).sum()
    g4 = 3 * m4 * m0 * m0 + 6 * m2 * m2 * m0 - 2 * c * 3 * m2 * m0 * m0 + c * c * mass3
    # psi(v) psi(v') = sum_{a, b in {v1^2, v2^2, v3^2, -c}} a(v) b(v')
    facs = [(0, 1.0), (1, 1.0), (2, 1.0), (None, -c)]
    for ia, ca in facs:
        for ib, cb in facs:
            row = [None, None, None]
            for mode in range(3):
                left = pieces[0] if ia == mode else pieces[1]
                right = pieces[0] if ib == mode else pieces[1]
                row.append(outer(left, right))
            weights.append(nu * ca * cb / g4)
            mats.append(row)
    return weights, mats, v, w


def cfg3(seed: int = 0, Qx: int = 64, Qv: int = 64, r: int = 12):
    """Linearised BGK-type kinetic problem (BASELINE cfg3): rank-4 IC
    prod sin(k x_j + phi) * M(v) * (1 + a v + b (v^2 - 1)), k in {1, 2}, padded to r."""
    rng = np.random.default_rng(seed)
    weights, mats, v, w = bgk_operator_terms(Qx, Qv)
    x = 2 * np.pi * np.arange(Qx) / Qx
    M1 = maxwellian_1d(v)
    rank = 4
    kk = rng.integers(1, 3, size=(rank, 3))
    phi = rng.uniform(0, 2 * np.pi, size=(rank, 3))
    ab = rng.uniform(-0.5, 0.5, size=(rank, 3, 2))
    factors = []
    for j in range(3):
        factors.append(np.stack([np.sin(kk[t, j] * x + phi[t, j]) for t in range(rank)], axis=1))
    for i in range(3):
        factors.append(np.stack([M1 * (1 + ab[t, i, 0] * v + ab[t, i, 1] * (v * v - 1)) for t in range(rank)],
                                axis=1))
    pad = [1e-8 * rng.standard_normal((f.shape[0], r - rank)) for f in factors]
    factors = [np.hstack([f, p]) for f, p in zip(factors, pad)]
    specs = tuple([BasisSpec(Qx, np.pi, "collocation", lo=0.0)] * 3 + [BasisSpec(Qv, 6.0, "uniform")] * 3)
    return dict(specs=specs, factors=factors, weights=weights, mats=mats, dt=1e-3, steps=200, r=r, sweeps=10,
                lam=1e-10, v=v, w=w)


def cfg4(seed: int = 0, batch: int = 64, d: int = 8, Q: int = 128, k: int = 64):
    """Batch of HT tensors on balanced trees: leaves N(0,1) (Q x k), transfers N(0,1) (k x k x k), root k x k x 1."""
    rng = np.random.default_rng(seed)
    n_nodes = 2 * d - 1
    n_int = d - 1
    frames = rng.standard_normal((batch, d, Q, k))
    transfers = rng.standard_normal((batch, n_int, k, k, k))
    return dict(frames=frames, transfers=transfers, d=d, Q=Q, k=k, r_max=16, eps=0.0, n_nodes=n_nodes)


__all__ = ["cfg0", "cfg1", "cfg2", "cfg3", "cfg4", "bgk_operator_terms", "advection_ic", "advection_exact", "nodes", "ADV_A"]
