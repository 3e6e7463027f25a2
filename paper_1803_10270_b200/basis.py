"""One-dimensional bases: the reference's odd-Q complex Fourier Galerkin basis
(``basis.py``) plus the real nodal bases the BASELINE configs use.

The truncation kernels never touch the basis (ALS and hSVD
are basis-agnostic), so a spec only has to supply ``Q`` and the host-side
factor matrices of separable operators:

* ``kind="fourier"`` -- the reference basis on ``[-b, b]`` with odd ``Q``
  (basis.py:54-71).  Its factor matrices are complex (basis.py:168-187); the
  B200 path computes in real fp64, so operators over this basis are rejected
  by ``operators.apply`` (SURVEY.md 8(f) row f4 is the complex follow-up).
* ``kind="collocation"`` -- nodal values on the periodic grid
  ``lo + 2b j / Q`` (any ``Q``, even allowed) with the Fourier collocation
  derivative matrix (BASELINE configs 0, 2 and the x-modes of config 3).
* ``kind="uniform"`` -- nodal values on ``linspace(-b, b, Q)`` (velocity
  modes of config 3; only multiplication factors are defined).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

__all__ = ["quadrature_weights", "interpolation_weights", "BasisSpec", "FactorKind", "factor_matrix", "fourier_diff_matrix", "nodes"]


class FactorKind(enum.Enum):
    """One-dimensional factor of a separable operator term (basis.py:35-41)."""

    IDENTITY = "identity"
    DERIVATIVE = "derivative"
    COORD_MULTIPLY = "coord_multiply"
    COORD_TIMES_DERIVATIVE = "coord_times_derivative"


@dataclass(frozen=True)
class BasisSpec:
    Q: int
    b: float
    kind: str = "fourier"
    lo: float | None = None

    def __post_init__(self):
        if self.kind not in ("fourier", "collocation", "uniform"):
            raise ValueError(f"unknown basis kind {self.kind!r}")
        if self.Q < 1 or (self.kind == "fourier" and self.Q % 2 == 0):
            raise ValueError(f"Q must be a positive odd integer, got {self.Q}")
        if not self.b > 0:
            raise ValueError(f"b must be positive, got {self.b}")

    @property
    def modes(self) -> np.ndarray:
        half = (self.Q - 1) // 2
        return np.arange(-half, half + 1)


def nodes(spec: BasisSpec) -> np.ndarray:
    if spec.kind == "collocation":
        lo = -spec.b if spec.lo is None else spec.lo
        return lo + 2.0 * spec.b * np.arange(spec.Q) / spec.Q
    if spec.kind == "uniform":
        return np.linspace(-spec.b, spec.b, spec.Q)
    raise ValueError("the Fourier Galerkin basis has no nodes")


def fourier_diff_matrix(Q: int, length: float = 2 * np.pi) -> np.ndarray:
    """Periodic Fourier collocation first-derivative matrix (any Q >= 1).

    Even Q: D_ij = (1/2)(-1)^(i-j) cot((i-j)h/2); odd Q: (1/2)(-1)^(i-j) csc((i-j)h/2);
    h = 2 pi / Q, scaled by 2 pi / length.  Exact on trigonometric polynomials
    of degree < Q/2.
    """
    h = 2 * np.pi / Q
    i = np.arange(Q)
    diff = i[:, None] - i[None, :]
    D = np.zeros((Q, Q))
    off = diff != 0
    sign = np.where(diff % 2 == 0, 1.0, -1.0)
    if Q % 2 == 0:
        D[off] = 0.5 * sign[off] / np.tan(diff[off] * h / 2)
    else:
        D[off] = 0.5 * sign[off] / np.sin(diff[off] * h / 2)
    return D * (2 * np.pi / length)


def _galerkin_factor(spec: BasisSpec, kind: FactorKind) -> np.ndarray:
    """basis.py:168-187 (closed forms of basis.py:97-156), complex."""
    s = spec.modes
    if kind is FactorKind.IDENTITY:
        return np.eye(spec.Q, dtype=complex)
    D = np.diag(1j * np.pi * s / spec.b)
    if kind is FactorKind.DERIVATIVE:
        return D
    m = s[None, :] - s[:, None]
    sign = np.where(m % 2 == 0, 1.0, -1.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        coord = np.where(m == 0, 0.0 + 0.0j, -1j * spec.b * sign / (np.pi * m))
    if kind is FactorKind.COORD_MULTIPLY:
        return coord
    return coord @ D


def factor_matrix(spec: BasisSpec, kind: FactorKind) -> np.ndarray:
    """Dense (Q, Q) matrix of a factor action in the given basis."""
    if spec.kind == "fourier":
        return _galerkin_factor(spec, kind)
    if kind is FactorKind.IDENTITY:
        return np.eye(spec.Q)
    x = nodes(spec)
    if spec.kind == "uniform":
        if kind is FactorKind.COORD_MULTIPLY:
            return np.diag(x)
        raise ValueError("uniform (non-periodic) grids define only multiplication factors")
    D = fourier_diff_matrix(spec.Q, 2.0 * spec.b)
    if kind is FactorKind.DERIVATIVE:
        return D
    if kind is FactorKind.COORD_MULTIPLY:
        return np.diag(x)
    return np.diag(x) @ D


def quadrature_weights(spec: BasisSpec, p: int) -> np.ndarray:
    """Nodal counterpart of ``integration_weights`` (basis.py:159-165): weights w with
    w . f ~ Int z^p f(z) dz for nodal values f.  Periodic collocation grids use the
    trapezoid rule (spectrally accurate for smooth periodic integrands), uniform
    grids on [-b, b] the composite trapezoid rule with half end weights."""
    if p not in (0, 1, 2):
        raise ValueError("moment power must be 0, 1 or 2")
    if spec.kind == "fourier":
        raise ValueError("the complex Galerkin basis is outside the real-fp64 device path")
    x = nodes(spec)
    if spec.kind == "collocation":
        w = np.full(spec.Q, 2.0 * spec.b / spec.Q)
    else:
        h = 2.0 * spec.b / (spec.Q - 1) if spec.Q > 1 else 2.0 * spec.b
        w = np.full(spec.Q, h)
        if spec.Q > 1:
            w[0] = w[-1] = 0.5 * h
    return w * x ** p


def interpolation_weights(spec: BasisSpec, z) -> np.ndarray:
    """Rows v(z) with v(z) . f = the grid function's interpolant at z (the nodal
    counterpart of ``eval_basis``, basis.py:74-94): trigonometric interpolation on
    periodic collocation grids (band-limited, Nyquist mode as a cosine), piecewise
    linear on uniform grids."""
    z = np.atleast_1d(np.asarray(z, dtype=float))
    if spec.kind == "fourier":
        raise ValueError("the complex Galerkin basis is outside the real-fp64 device path")
    Q = spec.Q
    x = nodes(spec)
    if spec.kind == "uniform":
        out = np.zeros((z.size, Q))
        if Q == 1:
            out[:, 0] = 1.0
            return out
        h = x[1] - x[0]
        t = np.clip((z - x[0]) / h, 0.0, Q - 1.0)
        i = np.minimum(np.floor(t).astype(int), Q - 2)
        fr = t - i
        out[np.arange(z.size), i] = 1.0 - fr
        out[np.arange(z.size), i + 1] = fr
        return out
    L = 2.0 * spec.b
    theta = 2.0 * np.pi * (z[:, None] - x[None, :]) / L          # (m, Q)
    kmax = (Q - 1) // 2
    acc = np.ones_like(theta)
    for m in range(1, kmax + 1):
        acc += 2.0 * np.cos(m * theta)
    if Q % 2 == 0:
        acc += np.cos((Q // 2) * theta)
    return acc / Q
