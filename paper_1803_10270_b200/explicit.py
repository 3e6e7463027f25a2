"""Two-step Adams-Bashforth integration with rank reduction (mirror of
``tensorpde/explicit.py``).

``recipe="split"`` is the reference recipe verbatim (explicit.py:85-103):
reduce the difference, the operator image and the update separately, with the
reference's adaptive ``rank_reduce_als`` (CP) or ``ht.truncate`` (HT).

``recipe="fused"`` is the SURVEY 8(a) row A10 recipe the BASELINE configs 0/3
use: the same AB2 / RK2 arithmetic, one fixed-rank ALS truncation per update,
warm-started from the previous solution:
    f2 = T(f1 + dt/2 L(3 f1 - f0); init=f1)
The target is assembled on the device by the K1 apply kernel directly into one
buffer (no host round trips), and ``run`` drives a whole trajectory with a
single status check at the end.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass, field

import torch

from . import cp, ht, operators
from .cp import ALSApproxConfig, CPTensor, inner_product, rank_reduce_als
from .ht import HTTensor
from .operators import SeparableOperator

__all__ = ["ExplicitConfig", "ReductionRecord", "ab2_step", "startup_step", "tensor_rank", "run"]

# captured AB2 steps of explicit.run, per operator (weak: dropped with the operator)
_GRAPHS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


@dataclass
class ExplicitConfig:
    dt: float
    r_max: int
    eps_rank: float = 1e-10
    format: str = "cp"          # "cp" or "ht"
    startup: str = "rk2"
    als: ALSApproxConfig = field(default_factory=ALSApproxConfig)
    recipe: str = "split"       # "split" (reference) or "fused" (BASELINE cfg0/cfg3)
    draws: str = "auto"         # rank_reduce_als random terms: "reference" = complex (cp.py:356-360)

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.r_max < 1:
            raise ValueError("rank cap must be at least 1")
        if self.format not in ("cp", "ht"):
            raise ValueError(f"unknown format {self.format!r}")
        if self.startup != "rk2":
            raise ValueError(f"unknown startup rule {self.startup!r}")
        if self.recipe not in ("split", "fused"):
            raise ValueError(f"unknown recipe {self.recipe!r}")
        if self.draws not in ("auto", "reference"):
            raise ValueError(f"unknown draws {self.draws!r}")


@dataclass
class ReductionRecord:
    stage: str
    rank_before: int
    rank_after: int
    error: float


def tensor_rank(f) -> int:
    return f.rank if isinstance(f, CPTensor) else f.max_rank


def _gap(f, red) -> float:
    g = inner_product(f, f) - 2.0 * inner_product(red, f) + inner_product(red, red)
    return float(max(g, 0.0) ** 0.5)


def _reduce(f, config: ExplicitConfig, stage: str, log, init=None):
    """explicit.py:56-74 (+ the fused warm-started fixed-rank truncation)."""
    if tensor_rank(f) <= config.r_max:
        if log is not None:
            log.append(ReductionRecord(stage, tensor_rank(f), tensor_rank(f), 0.0))
        return f
    if isinstance(f, CPTensor):
        if config.recipe == "fused" and init is not None and init.rank == config.r_max:
            red = cp.cp_approx_als(f, config.r_max, config.als, init=init)
        else:
            red = rank_reduce_als(f, config.r_max, config.eps_rank, config.als, draws=config.draws)
        if log is not None:
            log.append(ReductionRecord(stage, f.rank, red.rank, _gap(f, red)))
        return red
    red, est = ht.truncate(f, config.r_max, config.eps_rank)
    if log is not None:
        log.append(ReductionRecord(stage, f.max_rank, red.max_rank, est))
    return red


def _ops(f):
    if isinstance(f, CPTensor):
        return cp.add, cp.scale, operators.apply
    if isinstance(f, HTTensor):
        return ht.add, ht.scale, ht.apply_operator
    raise TypeError(f"unsupported tensor type {type(f).__name__}")


def ab2_target(f_n: CPTensor, f_n1: CPTensor, L: SeparableOperator, dt: float) -> CPTensor:
    """Exact AB2 update ``f1 + dt/2 L(3 f1 - f0)`` in one device buffer:
    columns [f1 | term-major L(w)], w = [3 f1 | -f0] (explicit.py:91-93 arithmetic)."""
    w = cp.concat(f_n1.specs, [(f_n1, 3.0), (f_n, -1.0)])
    out = cp.empty_cp(f_n1.specs, f_n1.rank + L.n_terms * w.rank, f_n1.data.device)
    cp._apply_raw(f_n1, [[None] * f_n1.ndim], [1.0], 1.0, None, out, 0)
    operators.apply_into(L, w, out, f_n1.rank, 0.5 * dt)
    return out


def _euler_target(f0: CPTensor, g: CPTensor, L: SeparableOperator, h: float) -> CPTensor:
    """``f0 + h L g`` in one device buffer: [f0 | term-major h L(g)]."""
    out = cp.empty_cp(f0.specs, f0.rank + L.n_terms * g.rank, f0.data.device)
    cp._apply_raw(f0, [[None] * f0.ndim], [1.0], 1.0, None, out, 0)
    operators.apply_into(L, g, out, f0.rank, h)
    return out


def ab2_step(f_n, f_n1, L: SeparableOperator, config: ExplicitConfig, log: list | None = None):
    """Advance to f_{n+2} given the two previous states (explicit.py:85-93)."""
    if type(f_n) is not type(f_n1):
        raise TypeError("both states must use the same tensor format")
    if config.recipe == "fused" and isinstance(f_n1, CPTensor):
        return _reduce(ab2_target(f_n, f_n1, L, config.dt), config, "update", log, init=f_n1)
    add, scale, apply_op = _ops(f_n1)
    w = _reduce(add(scale(f_n1, 3.0), scale(f_n, -1.0)), config, "difference", log)
    lw = _reduce(apply_op(L, w), config, "operator", log)
    return _reduce(add(f_n1, scale(lw, 0.5 * config.dt)), config, "update", log)


def startup_step(f_0, L: SeparableOperator, config: ExplicitConfig, log: list | None = None):
    """One explicit midpoint step to seed the two-step scheme (explicit.py:96-103)."""
    if config.recipe == "fused" and isinstance(f_0, CPTensor):
        half = _reduce(_euler_target(f_0, f_0, L, 0.5 * config.dt), config, "startup-half", log, init=f_0)
        return _reduce(_euler_target(f_0, half, L, config.dt), config, "startup-update", log, init=f_0)
    add, scale, apply_op = _ops(f_0)
    lf = _reduce(apply_op(L, f_0), config, "startup-operator", log)
    half = _reduce(add(f_0, scale(lf, 0.5 * config.dt)), config, "startup-half", log)
    lh = _reduce(apply_op(L, half), config, "startup-operator", log)
    return _reduce(add(f_0, scale(lh, config.dt)), config, "startup-update", log)


def run(f0: CPTensor, L: SeparableOperator, config: ExplicitConfig, steps: int, callback=None,
        graph: bool = True) -> CPTensor:
    """Fused-recipe CP trajectory (RK2 startup + AB2), fully stream-ordered:
    one fused-ALS launch per update, status words gathered on the device and
    checked once at the end (no per-step host synchronisation).

    ``graph``: after the startup and one eager AB2 step, one AB2 step (target
    assembly, truncation, state rotation) is captured into a CUDA graph and
    replayed for the remaining steps -- no per-step host launch overhead.  The
    replayed kernels are the eager ones on the same data: results are bitwise
    identical to ``graph=False``."""
    if config.recipe != "fused" or not isinstance(f0, CPTensor):
        prev, cur = f0, startup_step(f0, L, config)
        for n in range(2, steps + 1):
            prev, cur = cur, ab2_step(prev, cur, L, config)
        return cur
    r = config.r_max
    if f0.rank != r:
        raise ValueError(f"fused recipe needs the initial state at rank r_max={r}, got {f0.rank}")
    dev = f0.data.device
    infos = torch.zeros((max(steps, 1) + 1, 2), dtype=torch.int32, device=dev)

    def trunc(target: CPTensor, init: CPTensor, slot: int) -> CPTensor:
        if target.rank <= r:
            return target
        out = init.copy()
        cp._als_device(target, out.data, r, config.als, None, infos[slot])
        return out

    half = trunc(_euler_target(f0, f0, L, 0.5 * config.dt), f0, 0)
    cur = trunc(_euler_target(f0, half, L, config.dt), f0, 1)
    prev = f0
    if callback:
        callback(1, cur)
    use_graph = graph and callback is None and dev.type == "cuda" and steps >= 4 and \
        L.n_terms * 2 * r + r > r
    n_eager = 2 if use_graph else steps
    for n in range(2, n_eager + 1):
        nxt = trunc(ab2_target(prev, cur, L, config.dt), cur, n)
        prev, cur = cur, nxt
        if callback:
            callback(n, cur)
    if use_graph:
        # one captured AB2 step on static state buffers (rotated in place by the step),
        # cached per (operator, shapes, step configuration): later runs copy their
        # states in and replay -- every kernel of every step still executes
        a = config.als
        key = (tuple(cur.specs), r, float(config.dt), a.max_sweeps, float(a.tol), float(a.stall), a.seed,
               a.reg, a.grid, str(cur.data.dtype), dev.index)
        per_op = _GRAPHS.setdefault(L, {})
        hit = per_op.get(key)
        if hit is None:
            pbuf, cbuf = prev.data.clone(), cur.data.clone()
            slot = torch.zeros(2, dtype=torch.int32, device=dev)
            agg = torch.zeros(2, dtype=torch.int32, device=dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                P = CPTensor(cur.specs, data=pbuf, rank=r)
                C = CPTensor(cur.specs, data=cbuf, rank=r)
                tgt = ab2_target(P, C, L, config.dt)
                nxt = cbuf.clone()
                cp._als_device(tgt, nxt, r, config.als, None, slot)
                agg.bitwise_or_(slot)
                pbuf.copy_(cbuf)
                cbuf.copy_(nxt)
            hit = per_op[key] = (g, pbuf, cbuf, agg)
        g, pbuf, cbuf, agg = hit
        pbuf.copy_(prev.data)
        cbuf.copy_(cur.data)
        agg.zero_()
        for _ in range(n_eager + 1, steps + 1):
            g.replay()
        infos[n_eager + 1].copy_(agg)
        cur = CPTensor(cur.specs, data=cbuf.clone(), rank=r)
    bad = int(infos[:, 0].max().item())
    if bad & 2:
        raise cp.ConditioningError("normal equations produced non-finite coefficients")
    if bad & 1:
        raise cp.ConditioningError("regularised normal equations are not positive definite")
    _ = math
    return cur
