"""TEST INFRASTRUCTURE ONLY -- restatement of ``tensorpde/explicit.py`` (AB2 + RK2 startup).

Two recipes:

* ``split`` -- the reference recipe verbatim (explicit.py:85-103): reduce the
  difference, the operator image and the update separately;
* ``fused`` -- the SURVEY 8(a) row A10 recipe used by BASELINE configs 0/3: the
  same AB2/RK2 arithmetic, one truncation per update, warm-started from the
  previous solution: ``f2 = T(f1 + dt/2 L(3 f1 - f0); init=f1)``.

``reduce(target, init)`` is the truncation callback; the no-op rule of
``_reduce`` (explicit.py:56-61: leave tensors at or under the cap untouched)
is applied here, before the callback.
"""

from __future__ import annotations

from . import cp_als
from .operators import apply


def _noop_or(reduce, r_max):
    def red(t, init):
        if t[0].shape[1] <= r_max:           # explicit.py:58-61
            return t
        return reduce(t, init)
    return red


def ab2_split(f0, f1, weights, mats, dt, r_max, reduce):
    """explicit.py:85-93."""
    red = _noop_or(reduce, r_max)
    w = red(cp_als.add(cp_als.scale(f1, 3.0), cp_als.scale(f0, -1.0)), None)
    lw = red(apply(weights, mats, w), None)
    return red(cp_als.add(f1, cp_als.scale(lw, 0.5 * dt)), None)


def startup_split(f0, weights, mats, dt, r_max, reduce):
    """explicit.py:96-103 (explicit midpoint)."""
    red = _noop_or(reduce, r_max)
    lf = red(apply(weights, mats, f0), None)
    half = red(cp_als.add(f0, cp_als.scale(lf, 0.5 * dt)), None)
    lh = red(apply(weights, mats, half), None)
    return red(cp_als.add(f0, cp_als.scale(lh, dt)), None)


def ab2_target(f0, f1, weights, mats, dt):
    """The exact (unreduced) AB2 update ``f1 + dt/2 L(3 f1 - f0)`` in term order [f1 | L-blocks]."""
    w = cp_als.add(cp_als.scale(f1, 3.0), cp_als.scale(f0, -1.0))
    return cp_als.add(f1, cp_als.scale(apply(weights, mats, w), 0.5 * dt))


def ab2_fused(f0, f1, weights, mats, dt, r_max, reduce):
    red = _noop_or(reduce, r_max)
    return red(ab2_target(f0, f1, weights, mats, dt), f1)


def startup_fused(f0, weights, mats, dt, r_max, reduce):
    red = _noop_or(reduce, r_max)
    half = red(cp_als.add(f0, cp_als.scale(apply(weights, mats, f0), 0.5 * dt)), f0)
    return red(cp_als.add(f0, cp_als.scale(apply(weights, mats, half), dt)), f0)


def warm_als_reducer(sweeps, lam):
    """Fixed-rank ALS warm-started from ``init`` (BASELINE cfg0/cfg3 truncation)."""
    def reduce(t, init):
        return cp_als.als(t, init, sweeps, lam=lam)
    return reduce


def run_fused(f0, weights, mats, dt, r, steps, sweeps, lam, callback=None):
    """``steps`` time steps: one RK2 startup, then AB2 (BASELINE cfg0/cfg3 trajectory)."""
    red = warm_als_reducer(sweeps, lam)
    prev, cur = f0, startup_fused(f0, weights, mats, dt, r, red)
    if callback:
        callback(1, cur)
    for n in range(2, steps + 1):
        prev, cur = cur, ab2_fused(prev, cur, weights, mats, dt, r, red)
        if callback:
            callback(n, cur)
    return cur
