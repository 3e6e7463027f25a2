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


def cfg4(seed: int = 0, batch: int = 64, d: int = 8, Q: int = 128, k: int = 64):
    """Batch of HT tensors on balanced trees: leaves N(0,1) (Q x k), transfers N(0,1) (k x k x k), root k x k x 1."""
    rng = np.random.default_rng(seed)
    n_nodes = 2 * d - 1
    n_int = d - 1
    frames = rng.standard_normal((batch, d, Q, k))
    transfers = rng.standard_normal((batch, n_int, k, k, k))
    return dict(frames=frames, transfers=transfers, d=d, Q=Q, k=k, r_max=16, eps=0.0, n_nodes=n_nodes)


__all__ = ["cfg0", "cfg1", "cfg2", "cfg4", "advection_ic", "advection_exact", "nodes", "ADV_A"]
