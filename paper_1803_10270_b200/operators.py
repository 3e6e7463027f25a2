"""Separable linear operators (mirror of ``tensorpde/operators.py``).

An operator is ``sum_t w_t prod_k E^t_k``.  Beyond the reference's
``FactorKind`` entries (operators.py:28-45), a factor may be a dense
``(Q_k, Q_k)`` matrix or ``None`` (identity) -- the extension SURVEY 8(a) row
A4 requires for the BASELINE collocation operators (Fourier D, diag(v),
rank-1 moment projectors).  ``apply`` runs the sm_100a K1 kernel and writes
the term-major result (operators.py:48-62) in one launch; complex factor
matrices (the reference's Fourier Galerkin basis) or complex weights run the
complex128 kernel and give a complex result.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .basis import BasisSpec, FactorKind, factor_matrix
from .cp import CPTensor, _apply_raw, empty_cp

__all__ = ["SeparableOperator", "CrankNicolsonPair", "apply", "apply_into", "crank_nicolson_pair",
           "implicit_euler_pair", "advection_operator"]


@dataclass(frozen=True, eq=False)
class SeparableOperator:
    specs: tuple
    weights: tuple
    factors: tuple  # [term][dimension]: FactorKind | ndarray | None

    def __post_init__(self):
        if len(self.weights) != len(self.factors):
            raise ValueError("one weight per term required")
        if not self.factors:
            raise ValueError("operator needs at least one term")
        for row in self.factors:
            if len(row) != len(self.specs):
                raise ValueError("every term must assign a factor to every dimension")

    @property
    def n_terms(self) -> int:
        return len(self.weights)


_TABLES: "weakref.WeakKeyDictionary[SeparableOperator, tuple]" = weakref.WeakKeyDictionary()


def _is_identity(m) -> bool:
    return m is None or m is FactorKind.IDENTITY


def _real_weight(w) -> float:
    w = complex(w)
    if w.imag != 0:
        raise ValueError("complex operator weights are not supported by the real-fp64 implicit path")
    return w.real


def _weight(w):
    """Real weights stay float (real kernel); complex ones select the complex128 path."""
    w = complex(w)
    return w if w.imag != 0 else w.real


def dense_factor(spec: BasisSpec, m) -> np.ndarray | None:
    """Resolve a factor entry to a dense matrix (None = identity): float64 when
    real-valued, complex128 otherwise (Fourier Galerkin factors, basis.py:168-187)."""
    if _is_identity(m):
        return None
    if isinstance(m, FactorKind):
        m = factor_matrix(spec, m)
    m = np.asarray(m)
    if np.iscomplexobj(m):
        if np.any(m.imag != 0):
            if m.shape != (spec.Q, spec.Q):
                raise ValueError(f"factor matrix shape {m.shape} != ({spec.Q}, {spec.Q})")
            return np.ascontiguousarray(m, dtype=np.complex128)
        m = m.real
    if m.shape != (spec.Q, spec.Q):
        raise ValueError(f"factor matrix shape {m.shape} != ({spec.Q}, {spec.Q})")
    return np.ascontiguousarray(m, dtype=np.float64)


def device_tables(op: SeparableOperator, dev: torch.device):
    """Upload the distinct factor matrices once per operator: (mats, offsets, idx rows, weights)."""
    hit = _TABLES.get(op)
    if hit is not None and hit[0].device == dev:
        return hit
    mats, offs, rows, keys = [], [], [], {}
    off = 0
    for t, row in enumerate(op.factors):
        idx_row = []
        for k, m in enumerate(row):
            dm = dense_factor(op.specs[k], m)
            if dm is None:
                idx_row.append(None)
                continue
            key = (k, dm.tobytes())
            if key not in keys:
                keys[key] = len(offs)
                offs.append(off)
                mats.append(dm.reshape(-1))
                off += dm.size
            idx_row.append(keys[key])
        rows.append(idx_row)
    weights = [_weight(w) for w in op.weights]
    cplx = any(np.iscomplexobj(m) for m in mats) or any(isinstance(w, complex) for w in weights)
    dt = np.complex128 if cplx else np.float64
    buf = torch.as_tensor(np.concatenate([m.astype(dt) for m in mats]) if mats else np.zeros(1, dtype=dt)).to(dev)
    out = (buf, offs, rows, weights)
    _TABLES[op] = out
    return out


def is_complex(op: SeparableOperator) -> bool:
    """True when the operator needs the complex128 path (complex factors or weights)."""
    buf = device_tables(op, _lib.device())[0]
    return buf.is_complex()


def apply_into(op: SeparableOperator, f: CPTensor, out: CPTensor, col_off: int, scale=1.0) -> None:
    """Write ``scale * op(f)`` into columns [col_off, col_off + n_terms*rank) of ``out``."""
    if op.specs != f.specs:
        raise ValueError("operator and tensor live on different bases")
    buf, offs, rows, weights = device_tables(op, f.data.device)
    if (buf.is_complex() or f.is_complex) and not out.is_complex:
        raise ValueError("complex operator or tensor needs a complex128 output")
    _apply_raw(f, rows, weights, scale, buf, out, col_off, offs)


def apply(op: SeparableOperator, f: CPTensor) -> CPTensor:
    """Apply exactly; result rank ``n_terms * f.rank``, term-major (operators.py:48-62).
    Complex operator or tensor: complex128 result."""
    if op.specs != f.specs:
        raise ValueError("operator and tensor live on different bases")
    buf = device_tables(op, f.data.device)[0]
    cplx = buf.is_complex() or f.is_complex
    out = empty_cp(f.specs, op.n_terms * f.rank, f.data.device, torch.complex128 if cplx else torch.float64)
    apply_into(op, f, out, 0)
    return out


def advection_operator(a, specs) -> SeparableOperator:
    """``L = -sum_i a_i d/dx_i`` with one DERIVATIVE term per dimension (BASELINE cfg0/2)."""
    specs = tuple(specs)
    n = len(specs)
    rows = tuple(tuple(FactorKind.DERIVATIVE if k == i else FactorKind.IDENTITY for k in range(n))
                 for i in range(n))
    return SeparableOperator(specs, tuple(-float(x) for x in a), rows)


@dataclass(frozen=True, eq=False)
class CrankNicolsonPair:
    """``A = sum_e eta_e prod_k E^e_k`` and ``B = sum_e zeta_e prod_k E^e_k`` with a
    shared factor table (operators.py:110-136)."""

    specs: tuple
    dt: float
    eta: tuple
    zeta: tuple
    factors: tuple
    operator: SeparableOperator

    @property
    def n_terms(self) -> int:
        return len(self.eta)

    @property
    def A(self) -> SeparableOperator:
        return SeparableOperator(self.specs, self.eta, self.factors)

    @property
    def B(self) -> SeparableOperator:
        return SeparableOperator(self.specs, self.zeta, self.factors)


def _split_identity(L: SeparableOperator):
    n = len(L.specs)
    ident = tuple([FactorKind.IDENTITY] * n)
    rows, ws, w_id = [], [], 0.0
    for w, kinds in zip(L.weights, L.factors):
        if all(_is_identity(m) for m in kinds):
            w_id += _real_weight(w)
        else:
            rows.append(kinds)
            ws.append(_real_weight(w))
    return ident, rows, ws, w_id


def crank_nicolson_pair(L: SeparableOperator, dt: float) -> CrankNicolsonPair:
    """operators.py:139-155: identity terms folded into term 0."""
    if not dt > 0:
        raise ValueError(f"dt must be positive, got {dt}")
    ident, rows, ws, w_id = _split_identity(L)
    eta = [1.0 - 0.5 * dt * w_id] + [-0.5 * dt * w for w in ws]
    zeta = [1.0 + 0.5 * dt * w_id] + [0.5 * dt * w for w in ws]
    return CrankNicolsonPair(L.specs, float(dt), tuple(eta), tuple(zeta), tuple([ident] + rows), L)


def implicit_euler_pair(L: SeparableOperator, dt: float) -> CrankNicolsonPair:
    """``A = I - dt L``, ``B = I`` in the same pair layout (BASELINE cfg2)."""
    if not dt > 0:
        raise ValueError(f"dt must be positive, got {dt}")
    ident, rows, ws, w_id = _split_identity(L)
    eta = [1.0 - dt * w_id] + [-dt * w for w in ws]
    zeta = [1.0] + [0.0] * len(ws)
    return CrankNicolsonPair(L.specs, float(dt), tuple(eta), tuple(zeta), tuple([ident] + rows), L)
