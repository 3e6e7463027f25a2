"""Oracle (test infrastructure only): restatement of the reference diagnostics
(tensorpde/diagnostics.py) on numpy arrays, with the integration weights passed
in so the same formulas check the device contractions.  Pinned by
tests/golden/diagnostics.npz (values the reference itself produced)."""

from __future__ import annotations

import numpy as np


def contract(factors, weights) -> float:
    """diagnostics.py:60-64: sum_l prod_k (w_k @ F_k)[l]."""
    rows = np.ones(factors[0].shape[1], dtype=complex)
    for w, f in zip(weights, factors):
        rows = rows * (w @ f)
    return float(np.sum(rows).real)


def moments(factors, weights0, weights1, weights2, R: float, vol: float, vdims):
    """diagnostics.py:67-97 with weights[p][k] = Int z^p phi(z) for dimension k."""
    density = contract(factors, weights0) / vol
    flux = np.empty(3)
    energy = np.empty(3)
    for i, d in enumerate(vdims):
        w1 = list(weights0)
        w1[d] = weights1[d]
        flux[i] = contract(factors, w1) / vol
        w2 = list(weights0)
        w2[d] = weights2[d]
        energy[i] = contract(factors, w2) / vol
    velocity = flux / density
    centered = float(np.sum(energy)) - density * float(velocity @ velocity)
    return density, velocity, centered / (3.0 * R * density)


def nmae(x, y) -> float:
    """diagnostics.py:31-40."""
    x, y = np.asarray(x, dtype=float), np.asarray(y, dtype=float)
    return float(np.mean(np.abs(x - y)) / (np.max(x) - np.min(y)))


def fit_decay_rate(times, series, floor=None) -> float:
    """diagnostics.py:121-143."""
    times, series = np.asarray(times, dtype=float), np.asarray(series, dtype=float)
    keep = np.ones(series.size, dtype=bool) if floor is None else series >= 2.0 * floor
    return float(-np.polyfit(times[keep], np.log(series[keep]), 1)[0])
