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

from . import _lib, cp, ht, operators
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


def _fused_trunc(A: CPTensor, Ws, L: SeparableOperator, scale: float, init: CPTensor, r: int,
                 acfg: ALSApproxConfig, info) -> torch.Tensor | None:
    """Apply + truncation in ONE launch when the problem fits the one-CTA kernel
    (``tp_cp_als_recipe_f64``): the target [A | scale L(w)],
    w = [c0 W0 | c1 W1], is assembled inside the kernel from the states and the
    operator's matrices.  Returns the fitted factor buffer, or None when the fused
    path does not apply (the caller materialises the target)."""
    if (A.is_complex or any(w.is_complex for w, _ in Ws) or acfg.tol > 0 or acfg.stall > -math.inf or
            acfg.grid or L.n_terms > 64 or init.rank != r):
        return None
    buf, offs, rows, weights = operators.device_tables(L, A.data.device)
    if buf.is_complex() or any(isinstance(x, complex) for x in weights):
        return None
    rw = Ws[0][0].rank
    R = A.rank + L.n_terms * len(Ws) * rw
    Lb = _lib.lib()
    qs = _lib.int_array(A.qs)
    nbytes = Lb.tp_cp_als_ws_bytes(A.ndim, qs, R, r, 0)
    if nbytes == 0:
        return None
    ws = _lib.WORKSPACE.get(nbytes, A.data.device)
    U = init.data.clone()
    idx = [(-1 if m is None else int(m)) for row in rows for m in row]
    reg, mode = (cp._REG, 1) if acfg.reg is None else (float(acfg.reg), 0)
    W1 = Ws[1][0].data.data_ptr() if len(Ws) > 1 else None
    st = Lb.tp_cp_als_recipe_f64(A.ndim, qs, r, A.data.data_ptr(), A.rank, Ws[0][0].data.data_ptr(), float(Ws[0][1]),
                                 W1, float(Ws[1][1]) if len(Ws) > 1 else 0.0, rw, L.n_terms,
                                 _lib.double_array([scale * float(w) for w in weights]), _lib.int_array(idx),
                                 buf.data_ptr(), _lib.ll_array(offs), len(offs), U.data_ptr(), int(acfg.max_sweeps),
                                 reg, mode, info.data_ptr(), ws.data_ptr(), ws.numel(),
                                 _lib.stream_ptr(A.data.device))
    if st == _lib.TP_EUNSUPPORTED:
        return None
    _lib.check(st, "cp_approx_als (fused apply)")
    return U


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
        graph: bool = True, fused: bool = True) -> CPTensor:
    """Fused-recipe CP trajectory (RK2 startup + AB2), fully stream-ordered:
    one fused-ALS launch per update, status words gathered on the device and
    checked once at the end (no per-step host synchronisation).

    ``graph``: after the startup and one eager AB2 step, one AB2 step (target
    assembly, truncation, state rotation) is captured into a CUDA graph and
    replayed for the remaining steps -- no per-step host launch overhead.  The
    replayed kernels are the eager ones on the same data: results are bitwise
    identical to ``graph=False``.

    ``fused`` (default): when the problem fits the one-CTA kernel, every truncation is
    ONE launch that assembles its target [f1 | dt/2 L(3 f1 - f0)] from the two states and
    the operator's matrices (``tp_cp_als_recipe_f64``) -- L w is never
    materialised; bitwise equal to ``fused=False``."""
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

    # one launch per truncation with the target assembled in the kernel (f1) when it fits
    Uh = _fused_trunc(f0, [(f0, 1.0)], L, 0.5 * config.dt, f0, r, config.als, infos[0]) if fused else None
    fuse = Uh is not None

    def euler(a: CPTensor, g: CPTensor, h: float, init: CPTensor, slot: int) -> CPTensor:
        if fuse:
            U = _fused_trunc(a, [(g, 1.0)], L, h, init, r, config.als, infos[slot])
            return CPTensor(a.specs, data=U, rank=r)
        return trunc(_euler_target(a, g, L, h), init, slot)

    def ab2(p: CPTensor, c: CPTensor, slot: int) -> CPTensor:
        if fuse:
            U = _fused_trunc(c, [(c, 3.0), (p, -1.0)], L, 0.5 * config.dt, c, r, config.als, infos[slot])
            return CPTensor(c.specs, data=U, rank=r)
        return trunc(ab2_target(p, c, L, config.dt), c, slot)

    half = CPTensor(f0.specs, data=Uh, rank=r) if fuse else trunc(_euler_target(f0, f0, L, 0.5 * config.dt), f0, 0)
    cur = euler(f0, half, config.dt, f0, 1)
    prev = f0
    if callback:
        callback(1, cur)
    use_graph = graph and callback is None and dev.type == "cuda" and steps >= 4 and \
        L.n_terms * 2 * r + r > r
    n_eager = 2 if use_graph else steps
    for n in range(2, n_eager + 1):
        nxt = ab2(prev, cur, n)
        prev, cur = cur, nxt
        if callback:
            callback(n, cur)
    if use_graph:
        # one captured AB2 step on static state buffers (rotated in place by the step),
        # cached per (operator, shapes, step configuration): later runs copy their
        # states in and replay -- every kernel of every step still executes
        a = config.als
        key = (tuple(cur.specs), r, float(config.dt), a.max_sweeps, float(a.tol), float(a.stall), a.seed,
               a.reg, a.grid, str(cur.data.dtype), dev.index, fuse)
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
                if fuse:
                    nxt = _fused_trunc(C, [(C, 3.0), (P, -1.0)], L, 0.5 * config.dt, C, r, config.als, slot)
                else:
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
    return cur
