"""Canonical (CP) tensors on the device and alternating least squares.

Drop-in mirror of the reference ``tensorpde/cp.py``.  A rank-``R`` tensor over
``d`` specs is ONE contiguous fp64 device buffer; mode ``k`` is the row-major
``(Q_k, R)`` block at element offset ``R * sum_{k'<k} Q_k'`` -- exactly the
reference's ``factors[k]`` array (cp.py:43-59), stacked mode-major.  Scalars
live in mode 0 (cp.py:1-12).  Real-valued data runs in real fp64 (the
BASELINE configs are real; the reference's complex128 agrees to ~1e-15 on real
data).  Complex data (the reference's Fourier Galerkin basis,
complex random initial terms) runs in complex128 through the ``*_c128``
kernels, the reference's own arithmetic.  All compute
runs through the sm_100a C-ABI library; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ConditioningError
from .basis import BasisSpec

__all__ = [
    "CPTensor", "ALSApproxConfig", "ConditioningError", "add", "scale", "inner_product", "norm",
    "random_cp", "pad_rank", "cp_approx_als", "check", "rank_reduce_als", "from_numpy_factors", "as_complex",
]


def _as_array(f, k):
    """Factor k as a CPU tensor: float64 when the values are real (also a complex
    array with zero imaginary part), complex128 otherwise."""
    if isinstance(f, torch.Tensor):
        f = f.detach().cpu()
        if f.is_complex():
            if torch.any(f.imag != 0):
                return f.to(torch.complex128)
            f = f.real
        return f.to(torch.float64)
    a = np.asarray(f)
    if np.iscomplexobj(a):
        if np.any(a.imag != 0):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.complex128))
        a = a.real
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64))


class CPTensor:
    """``CPTensor(specs, factors)`` validates like cp.py:47-59 and copies the
    factors into one device buffer (value semantics, like the reference's
    ``np.ascontiguousarray`` copy)."""

    __slots__ = ("specs", "data", "_rank", "pending_info")

    def __init__(self, specs, factors=None, *, data: torch.Tensor | None = None, rank: int | None = None):
        self.pending_info = None
        self.specs = tuple(specs)
        if data is not None:
            self.data = data
            self._rank = int(rank)
            return
        if factors is None or len(factors) != len(self.specs):
            raise ValueError("one factor matrix per dimension required")
        mats = [_as_array(f, k) for k, f in enumerate(factors)]
        if any(m.is_complex() for m in mats):   # one complex factor -> the whole tensor is complex128
            mats = [m.to(torch.complex128) for m in mats]
        ranks = {int(m.shape[1]) if m.dim() == 2 else -1 for m in mats}
        if len(ranks) != 1:
            raise ValueError(f"inconsistent ranks across dimensions: {ranks}")
        for k, (m, spec) in enumerate(zip(mats, self.specs)):
            if m.dim() != 2 or m.shape[0] != spec.Q:
                raise ValueError(f"dimension {k}: {m.shape[0]} rows != Q={spec.Q}")
        r = mats[0].shape[1]
        if r < 1:
            raise ValueError("rank must be at least 1")
        dev = _lib.device()
        self.data = torch.cat([m.reshape(-1) for m in mats]).to(dev)
        self._rank = int(r)

    # -- shape
    @property
    def is_complex(self) -> bool:
        return self.data.is_complex()

    @property
    def ndim(self) -> int:
        return len(self.specs)

    @property
    def rank(self) -> int:
        return self._rank

    @property
    def qs(self) -> tuple[int, ...]:
        return tuple(s.Q for s in self.specs)

    @property
    def factors(self) -> list[torch.Tensor]:
        """Per-mode ``(Q_k, R)`` views into the device buffer."""
        out, off = [], 0
        for q in self.qs:
            n = q * self._rank
            out.append(self.data[off:off + n].view(q, self._rank))
            off += n
        return out

    def copy(self) -> "CPTensor":
        return CPTensor(self.specs, data=self.data.clone(), rank=self._rank)

    def norm(self) -> float:
        return norm(self)

    def to_numpy(self) -> list[np.ndarray]:
        return [f.cpu().numpy().copy() for f in self.factors]

    def __repr__(self):
        return f"CPTensor(ndim={self.ndim}, Q={self.qs}, rank={self.rank}, device={self.data.device})"


def from_numpy_factors(specs, factors) -> CPTensor:
    return CPTensor(specs, factors)


def empty_cp(specs, rank: int, dev=None, dtype=torch.float64) -> CPTensor:
    n = sum(s.Q for s in specs) * rank
    return CPTensor(specs, data=torch.empty(n, dtype=dtype, device=dev or _lib.device()), rank=rank)


def as_complex(f: CPTensor) -> CPTensor:
    """complex128 copy of a real tensor (the reference's coercion, cp.py:59); complex tensors pass through."""
    if f.is_complex:
        return f
    return CPTensor(f.specs, data=f.data.to(torch.complex128), rank=f.rank)


def _is_cplx_scalar(c) -> bool:
    return isinstance(c, complex) and c.imag != 0


def _check_same_specs(f: CPTensor, g: CPTensor) -> None:
    if f.specs != g.specs:
        raise ValueError("operands live on different bases")


def concat(specs, parts) -> CPTensor:
    """Column concatenation of several (tensor, scale) parts in one device pass
    (cp.add / cp.scale, cp.py:98-108).  Scale goes into mode 0.  Any complex
    part or scale makes the result complex128."""
    cplx = any(t.is_complex or _is_cplx_scalar(complex(c)) for t, c in parts)
    parts = [(t, complex(c) if cplx else float(complex(c).real)) for t, c in parts]
    R = sum(t.rank for t, _ in parts)
    out = empty_cp(specs, R, parts[0][0].data.device, torch.complex128 if cplx else torch.float64)
    col = 0
    for t, c in parts:
        _apply_raw(t, [[None] * t.ndim], [1.0], c, None, out, col)
        col += t.rank
    return out


def add(f: CPTensor, g: CPTensor) -> CPTensor:
    """Exact sum; ranks add, g's terms follow f's (cp.py:98-101)."""
    _check_same_specs(f, g)
    return concat(f.specs, [(f, 1.0), (g, 1.0)])


def scale(f: CPTensor, c) -> CPTensor:
    """Scalar multiple folded into mode 0 (cp.py:104-108)."""
    return concat(f.specs, [(f, c)])


def _inner_device(f: CPTensor, g: CPTensor, out: torch.Tensor) -> None:
    L = _lib.lib()
    qs = _lib.int_array(f.qs)
    same = 1 if (f.data.data_ptr() == g.data.data_ptr() and f.rank == g.rank) else 0
    nbytes = L.tp_cp_inner_ws_bytes(f.ndim, qs, f.rank, g.rank)
    ws = _lib.WORKSPACE.get(nbytes, f.data.device)
    st = L.tp_cp_inner_f64(f.ndim, qs, f.rank, f.data.data_ptr(), g.rank, g.data.data_ptr(), same,
                           out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(f.data.device))
    _lib.check(st, "inner_product")


def _inner_device_c(f: CPTensor, g: CPTensor, out: torch.Tensor) -> None:
    L = _lib.lib()
    f, g = as_complex(f), as_complex(g)
    qs = _lib.int_array(f.qs)
    nbytes = L.tp_cp_inner_c128_ws_bytes(f.ndim, qs, f.rank, g.rank)
    ws = _lib.WORKSPACE.get(nbytes, f.data.device)
    st = L.tp_cp_inner_c128(f.ndim, qs, f.rank, f.data.data_ptr(), g.rank, g.data.data_ptr(), out.data_ptr(),
                            ws.data_ptr(), ws.numel(), _lib.stream_ptr(f.data.device))
    _lib.check(st, "inner_product")


def inner_product(f: CPTensor, g: CPTensor):
    """``<f, g> = sum_{l,n} prod_k (F_k^H G_k)[l, n]`` (cp.py:111-121), conjugate
    on f.  Real tensors: a Python float (the conjugation is the identity);
    complex tensors: a Python complex, like the reference."""
    _check_same_specs(f, g)
    if f.is_complex or g.is_complex:
        out = torch.empty(2, dtype=torch.float64, device=f.data.device)
        _inner_device_c(f, g, out)
        re, im = out.tolist()
        return complex(re, im)
    out = torch.empty(1, dtype=torch.float64, device=f.data.device)
    _inner_device(f, g, out)
    return float(out.item())


def norm(f: CPTensor) -> float:
    """cp.py:124-126."""
    return float(math.sqrt(max(complex(inner_product(f, f)).real, 0.0)))


def random_cp(specs, r: int, rng: np.random.Generator, complex_: bool = False) -> CPTensor:
    """Unit-normalised random terms (cp.py:129-136).  ``complex_=True`` draws
    exactly like the reference (real and imaginary N(0,1) parts from the same
    generator); the default real variant is used for real targets."""
    factors = []
    for spec in specs:
        if complex_:
            m = rng.standard_normal((spec.Q, r)) + 1j * rng.standard_normal((spec.Q, r))
        else:
            m = rng.standard_normal((spec.Q, r))
        m /= np.linalg.norm(m, axis=0, keepdims=True)
        factors.append(m)
    return CPTensor(tuple(specs), factors)


def pad_rank(f: CPTensor, r: int, rng: np.random.Generator, rel_scale: float = 1e-8) -> CPTensor:
    """cp.py:139-146 (complex random terms for a complex tensor)."""
    if r < f.rank:
        raise ValueError(f"cannot pad rank {f.rank} down to {r}")
    if r == f.rank:
        return f.copy()
    pad = scale(random_cp(f.specs, r - f.rank, rng, f.is_complex), rel_scale * max(norm(f), 1.0))
    return add(f, pad)


@dataclass
class ALSApproxConfig:
    """cp.py:150-163, plus:

    ``reg``   -- ``None``: the reference rule lambda = 1e-12 tr(H)/r (cp.py:166-173);
                 a float: fixed Tikhonov lambda (BASELINE: 1e-10).
    ``grid``  -- CTAs of the persistent ALS kernel (0 = library heuristic).
    ``max_sweeps/tol/stall/seed`` keep the reference meaning; ``stall=-inf``
    and ``tol=0`` run exactly ``max_sweeps`` sweeps.
    """

    max_sweeps: int = 200
    tol: float = 0.0
    stall: float = 1e-13
    seed: int = 0
    quad_points: int = 0
    reg: float | None = None
    grid: int = 0


_REG = 1e-12


def _als_device(target: CPTensor, U: torch.Tensor, r: int, cfg: ALSApproxConfig,
                trace_buf: torch.Tensor | None, info: torch.Tensor) -> None:
    """Launch the fused ALS on the current stream; U is overwritten in place
    (complex128 target and U: the one-CTA complex kernel)."""
    L = _lib.lib()
    qs = _lib.int_array(target.qs)
    d = target.ndim
    if target.is_complex:
        if not U.is_complex():
            raise ValueError("complex target needs a complex guess")
        nbytes = L.tp_cp_als_c128_ws_bytes(d, qs, target.rank, r)
        if nbytes == 0:
            raise ValueError(f"unsupported complex ALS size: d={d}, R={target.rank}, r={r} "
                             "(the complex path keeps the problem in one CTA's shared memory)")
        ws = _lib.WORKSPACE.get(nbytes, target.data.device)
        reg, mode = (_REG, 1) if cfg.reg is None else (float(cfg.reg), 0)
        st = L.tp_cp_als_c128(d, qs, target.rank, target.data.data_ptr(), r, U.data_ptr(), int(cfg.max_sweeps),
                              reg, mode, float(cfg.tol), float(cfg.stall),
                              trace_buf.data_ptr() if trace_buf is not None else None,
                              info.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(target.data.device))
        _lib.check(st, "cp_approx_als")
        return
    nbytes = L.tp_cp_als_ws_bytes(d, qs, target.rank, r, cfg.grid)
    if nbytes == 0:
        raise ValueError(f"unsupported ALS size: d={d}, R={target.rank}, r={r} (r <= 160, d <= 8)")
    ws = _lib.WORKSPACE.get(nbytes, target.data.device)
    reg, mode = (_REG, 1) if cfg.reg is None else (float(cfg.reg), 0)
    st = L.tp_cp_als_f64(d, qs, target.rank, target.data.data_ptr(), r, U.data_ptr(), int(cfg.max_sweeps),
                         reg, mode, float(cfg.tol), float(cfg.stall),
                         trace_buf.data_ptr() if trace_buf is not None else None,
                         info.data_ptr(), int(cfg.grid), ws.data_ptr(), ws.numel(),
                         _lib.stream_ptr(target.data.device))
    _lib.check(st, "cp_approx_als")


def als_plan(qs, R: int, r: int, grid: int = 0) -> dict:
    """Launch plan of the fused ALS kernel for these sizes (tp_cp_als_plan)."""
    out = (ctypes.c_int * 4)()
    st = _lib.lib().tp_cp_als_plan(len(qs), _lib.int_array(qs), R, r, grid, out)
    _lib.check(st, "als_plan")
    variant = {0: "als_persistent", 1: "als_cluster", 2: "als_small", 3: "als_persistent_cluster",
               5: "als_tiny8", 7: "als_generic", 8: "als_rows", 9: "als_w"}[out[0]]
    return {"kernel": variant, "ctas": out[1], "cluster": out[2], "smem_bytes": out[3]}


def _check_info(info: torch.Tensor) -> int:
    status, done = (int(v) for v in info.tolist())
    if status & 2:
        raise ConditioningError("normal equations produced non-finite coefficients")
    if status & 1:
        raise ConditioningError("regularised normal equations are not positive definite")
    if status & 4:
        raise RuntimeError("ALS kernel: a cooperating CTA never arrived (cross-CTA wait timed out)")
    return done


def cp_approx_als(target, r: int, config: ALSApproxConfig | None = None, *, specs=None,
                  init: CPTensor | None = None, trace: list | None = None, sync: bool = True) -> CPTensor:
    """Fit a rank-``r`` CP tensor to ``target`` by Gauss-Seidel ALS (cp.py:266-334).

    One call = one launch of the persistent fused ALS kernel (all sweeps).
    Callable targets (cp.py:212-263, quadrature projection) are out of the
    hot-path scope and raise ``NotImplementedError``.

    ``sync=False`` (B200 extension, pipelined callers): the status word is not
    read back; the result carries it and ``check(result)`` raises the reference's
    ConditioningError later (no host round trip per call).  Incompatible with
    ``trace``.
    """
    cfg = config or ALSApproxConfig()
    if not isinstance(target, CPTensor):
        if specs is None:
            raise ValueError("callable targets require specs")
        raise NotImplementedError("callable (quadrature) targets are outside the B200 hot path")
    specs = target.specs
    rng = np.random.default_rng(cfg.seed)
    guess = init.copy() if init is not None else random_cp(specs, r, rng, target.is_complex)
    if guess.rank != r or guess.specs != tuple(specs):
        raise ValueError("init shape does not match the requested fit")
    if target.is_complex or guess.is_complex:   # the reference's complex128 arithmetic
        target, guess = as_complex(target), as_complex(guess).copy()
    if not sync and trace is not None:
        raise ValueError("trace needs sync=True")
    dev = target.data.device
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    tb = torch.zeros(max(cfg.max_sweeps, 1), dtype=torch.float64, device=dev) if trace is not None else None
    _als_device(target, guess.data, r, cfg, tb, info)
    if not sync:
        guess.pending_info = info
        return guess
    done = _check_info(info)
    if trace is not None:
        trace.extend(tb[:done].tolist())
    return guess


def check(result: CPTensor) -> CPTensor:
    """Raise the deferred status of a ``cp_approx_als(..., sync=False)`` result."""
    info = result.pending_info
    if info is not None:
        _check_info(info)
        result.pending_info = None
    return result


def _relative_error(f: CPTensor, g: CPTensor, nf: float) -> float:
    """Gram-identity error as in cp.py:369-375 (what the reference's adaptive loop uses)."""
    d = (complex(inner_product(f, f)).real - 2.0 * complex(inner_product(g, f)).real
         + complex(inner_product(g, g)).real)
    return float(math.sqrt(max(d, 0.0)) / nf)


def rank_reduce_als(f: CPTensor, r_target: int, eps: float, config: ALSApproxConfig | None = None, *,
                    draws: str = "auto") -> CPTensor:
    """Adaptive rank 1..r_target, warm start + one fresh random term (cp.py:337-366).

    ``draws="reference"``: the reference's complex random terms from the same generator
    sequence for every target (real targets then fit in complex128, exactly as the
    reference does: its result is complex).  ``draws="auto"`` (default): complex draws
    for complex targets, real N(0,1) draws for real targets (the real fp64 kernels; a
    documented deviation)."""
    if r_target < 1:
        raise ValueError("target rank must be at least 1")
    if draws not in ("auto", "reference"):
        raise ValueError(f"draws must be 'auto' or 'reference', not {draws!r}")
    cfg = config or ALSApproxConfig()
    nf = norm(f)
    cz = f.is_complex or draws == "reference"
    if cz:
        f = as_complex(f)
    zero = CPTensor(f.specs, [np.zeros((s.Q, 1)) for s in f.specs])
    if cz:
        zero = as_complex(zero)
    if nf == 0.0:
        return zero
    rng = np.random.default_rng(cfg.seed)
    best, best_err = zero, 1.0
    guess = None
    for r in range(1, r_target + 1):
        init = random_cp(f.specs, 1, rng, cz) if guess is None else add(guess, random_cp(f.specs, 1, rng, cz))
        guess = cp_approx_als(f, r, cfg, init=init)
        err = _relative_error(f, guess, nf)
        if err < best_err:
            best, best_err = guess, err
        if err <= eps:
            return guess
    return best


# ---- operator apply into a preallocated target (shared with operators.py) ----

def _apply_raw(f: CPTensor, mat_rows, weights, scale_, mats_dev, out: CPTensor, col_off: int,
               mat_off=None) -> None:
    """Launch tp_cp_apply_f64 (or tp_cp_apply_c128 when ``out`` is complex128):
    mat_rows[t][k] is an int matrix index or None."""
    L = _lib.lib()
    d = f.ndim
    n_terms = len(weights)
    idx = []
    for row in mat_rows:
        idx.extend(-1 if m is None else int(m) for m in row)
    n_mats = 0 if mat_off is None else len(mat_off)
    if out.is_complex:
        f = as_complex(f)
        if mats_dev is not None and not mats_dev.is_complex():
            mats_dev = mats_dev.to(torch.complex128)
        w = []
        for x in weights:
            x = complex(x)
            w += [x.real, x.imag]
        sc = complex(scale_)
        st = L.tp_cp_apply_c128(d, _lib.int_array(f.qs), f.rank, f.data.data_ptr(), n_terms, _lib.double_array(w),
                                sc.real, sc.imag, _lib.int_array(idx),
                                None if mats_dev is None else mats_dev.data_ptr(),
                                None if mat_off is None else _lib.ll_array(mat_off), n_mats,
                                out.data.data_ptr(), out.rank, int(col_off), _lib.stream_ptr(f.data.device))
        _lib.check(st, "apply")
        return
    scale_ = complex(scale_).real
    st = L.tp_cp_apply_f64(d, _lib.int_array(f.qs), f.rank, f.data.data_ptr(), n_terms,
                           _lib.double_array(weights), float(scale_), _lib.int_array(idx),
                           None if mats_dev is None else mats_dev.data_ptr(),
                           None if mat_off is None else _lib.ll_array(mat_off), n_mats,
                           out.data.data_ptr(), out.rank, int(col_off), _lib.stream_ptr(f.data.device))
    _lib.check(st, "apply")

