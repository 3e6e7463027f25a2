"""TEST INFRASTRUCTURE ONLY -- restatement of ``operators.apply`` with dense factor matrices.

``factors[q][k]`` is either ``None`` (identity) or a dense ``(Q_k, Q_k)`` matrix;
this is shim S4 of SURVEY.md 8(c): the reference ``apply`` (operators.py:48-62) with ``factor_matrix``
replaced by an explicit matrix.
"""

from __future__ import annotations

import numpy as np


def apply(weights, factors, f):
    """Term-major output, weight in mode 0, identity factors copied (operators.py:48-62)."""
    d = len(f)
    blocks = [[] for _ in range(d)]
    for w, mats in zip(weights, factors):
        for k in range(d):
            col = f[k].copy() if mats[k] is None else mats[k] @ f[k]
            if k == 0:
                col = col * w
            blocks[k].append(col)
    return [np.hstack(cols) for cols in blocks]


def dense_matrix(weights, factors, qs):
    """Kronecker sum of the operator (reference tests/oracles.py:120-136 pattern)."""
    n = int(np.prod(qs))
    out = None
    for w, mats in zip(weights, factors):
        term = np.array([[1.0]])
        for q, m in zip(qs, mats):
            term = np.kron(term, np.eye(q) if m is None else m)
        out = w * term if out is None else out + w * term
    return out if out is not None else np.zeros((n, n))
