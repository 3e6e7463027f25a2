"""TEST INFRASTRUCTURE ONLY -- restatement of ``tensorpde/ht.py`` (HT format + hSVD truncation).

An HT tensor here is ``(nodes, frames, transfers)``: ``nodes`` a list of
``(dims, parent, left, right)`` tuples in the reference preorder
(ht.py:55-98), ``frames[i]`` a ``(Q, r_i)`` leaf basis, ``transfers[i]`` an
``(r_left, r_right, r_i)`` interior transfer tensor (root rank 1).
"""

from __future__ import annotations

import numpy as np


def balanced_tree(ndim):
    """ht.py:79-98: split each run in half, left child takes the floor; preorder indices."""
    nodes = []

    def build(dims, parent):
        idx = len(nodes)
        nodes.append(None)
        if len(dims) == 1:
            nodes[idx] = (dims, parent, -1, -1)
        else:
            half = len(dims) // 2
            left = build(dims[:half], idx)
            right = build(dims[half:], idx)
            nodes[idx] = (dims, parent, left, right)
        return idx

    build(tuple(range(ndim)), -1)
    return nodes


def is_leaf(node):
    return node[2] < 0


def from_cp(factors, nodes=None):
    """ht.py:165-186: exact conversion with diagonal transfers."""
    nodes = nodes or balanced_tree(len(factors))
    r = factors[0].shape[1]
    dt = factors[0].dtype
    frames = [None] * len(nodes)
    transfers = [None] * len(nodes)
    if len(factors) == 1:
        frames[0] = factors[0].sum(axis=1, keepdims=True)
        return nodes, frames, transfers
    diag = np.zeros((r, r, r), dtype=dt)
    diag[np.arange(r), np.arange(r), np.arange(r)] = 1.0
    for i, node in enumerate(nodes):
        if is_leaf(node):
            frames[i] = factors[node[0][0]].copy()
        elif i == 0:
            root = np.zeros((r, r, 1), dtype=dt)
            root[np.arange(r), np.arange(r), 0] = 1.0
            transfers[i] = root
        else:
            transfers[i] = diag.copy()
    return nodes, frames, transfers


def add(h1, h2):
    """ht.py:208-232: block-diagonal concatenation; the root keeps rank 1."""
    nodes, f1, t1 = h1
    _, f2, t2 = h2
    frames = [None] * len(nodes)
    transfers = [None] * len(nodes)
    if len(nodes) == 1:
        frames[0] = f1[0] + f2[0]
        return nodes, frames, transfers
    for i, node in enumerate(nodes):
        if is_leaf(node):
            frames[i] = np.hstack([f1[i], f2[i]])
            continue
        a, b = t1[i], t2[i]
        dt = np.result_type(a, b)
        if i == 0:
            blk = np.zeros((a.shape[0] + b.shape[0], a.shape[1] + b.shape[1], 1), dtype=dt)
            blk[:a.shape[0], :a.shape[1], 0] = a[:, :, 0]
            blk[a.shape[0]:, a.shape[1]:, 0] = b[:, :, 0]
        else:
            blk = np.zeros((a.shape[0] + b.shape[0], a.shape[1] + b.shape[1],
                            a.shape[2] + b.shape[2]), dtype=dt)
            blk[:a.shape[0], :a.shape[1], :a.shape[2]] = a
            blk[a.shape[0]:, a.shape[1]:, a.shape[2]:] = b
        transfers[i] = blk
    return nodes, frames, transfers


def scale(h, c):
    """ht.py:235-241: scalar folded into the root."""
    nodes, frames, transfers = h
    frames = [None if u is None else u.copy() for u in frames]
    transfers = [None if b is None else b.copy() for b in transfers]
    if is_leaf(nodes[0]):
        frames[0] = frames[0] * c
    else:
        transfers[0] = transfers[0] * c
    return nodes, frames, transfers


def inner_product(h1, h2):
    """ht.py:264-276: leaves-to-root Gram contraction, conjugate on h1."""
    nodes, f1, t1 = h1
    _, f2, t2 = h2
    grams = [None] * len(nodes)
    for i in reversed(range(len(nodes))):
        node = nodes[i]
        if is_leaf(node):
            grams[i] = f1[i].conj().T @ f2[i]
        else:
            grams[i] = np.einsum("abi,ac,bd,cdj->ij", t1[i].conj(), grams[node[2]],
                                 grams[node[3]], t2[i], optimize=True)
    return complex(grams[0][0, 0])


def _push_into_parent(nodes, transfers, idx, r):
    """ht.py:285-291."""
    parent = nodes[idx][1]
    bp = transfers[parent]
    if nodes[parent][2] == idx:
        transfers[parent] = np.einsum("ca,abi->cbi", r, bp, optimize=True)
    else:
        transfers[parent] = np.einsum("cb,abi->aci", r, bp, optimize=True)


def orthogonalize(h):
    """ht.py:294-310: leaves-to-root reduced QR, R pushed into the parent."""
    nodes, frames, transfers = h
    frames = [None if u is None else u.copy() for u in frames]
    transfers = [None if b is None else b.copy() for b in transfers]
    for i in reversed(range(1, len(nodes))):
        if is_leaf(nodes[i]):
            q, r = np.linalg.qr(frames[i])
            frames[i] = q
        else:
            b = transfers[i]
            q, r = np.linalg.qr(b.reshape(b.shape[0] * b.shape[1], b.shape[2]))
            transfers[i] = q.reshape(b.shape[0], b.shape[1], q.shape[1])
        _push_into_parent(nodes, transfers, i, r)
    return nodes, frames, transfers


def norm(h):
    """ht.py:279-282."""
    nodes, frames, transfers = h
    if is_leaf(nodes[0]):
        return float(np.linalg.norm(frames[0]))
    return float(np.linalg.norm(orthogonalize(h)[2][0]))


def keep_rule(lam_desc, r_max, budget):
    """ht.py:349-358: drop trailing eigenvalues while over the cap or within the budget."""
    keep = lam_desc.shape[0]
    tail = 0.0
    while keep > 1:
        step = max(float(lam_desc[keep - 1]), 0.0)
        if keep > r_max or tail + step <= budget:
            tail += step
            keep -= 1
        else:
            break
    return keep, tail


def truncate(h, r_max, eps, return_eigs=False):
    """ht.py:313-372: orthogonalize, root-to-leaves node Grams, eigh per node, project."""
    if r_max < 1:
        raise ValueError("rank cap must be at least 1")
    ortho = orthogonalize(h)
    nodes, oframes, otransfers = ortho
    if is_leaf(nodes[0]):
        return (ortho, 0.0, []) if return_eigs else (ortho, 0.0)
    total = float(np.linalg.norm(otransfers[0]))
    if total == 0.0:
        return (ortho, 0.0, []) if return_eigs else (ortho, 0.0)
    ndim = len(nodes[0][0])
    budget = (eps * total) ** 2 / max(2 * ndim - 3, 1)
    grams = [None] * len(nodes)
    grams[0] = np.eye(1, dtype=otransfers[0].dtype)
    for i, node in enumerate(nodes):
        if is_leaf(node):
            continue
        b = otransfers[i]
        grams[node[2]] = np.einsum("abi,ij,cbj->ac", b, grams[i], b.conj(), optimize=True)
        grams[node[3]] = np.einsum("abi,ij,acj->bc", b, grams[i], b.conj(), optimize=True)
    basis = [np.eye(1, dtype=otransfers[0].dtype)] * len(nodes)
    discarded = 0.0
    eigs = [None] * len(nodes)
    for i in range(1, len(nodes)):
        lam, w = np.linalg.eigh(0.5 * (grams[i] + grams[i].conj().T))
        lam, w = lam[::-1], w[:, ::-1]
        eigs[i] = lam.copy()
        keep, tail = keep_rule(lam, r_max, budget)
        discarded += tail
        basis[i] = w[:, :keep]
    frames = [None] * len(nodes)
    transfers = [None] * len(nodes)
    for i, node in enumerate(nodes):
        if is_leaf(node):
            frames[i] = oframes[i] @ basis[i]
        else:
            transfers[i] = np.einsum("abi,ac,bd,ie->cde", otransfers[i], basis[node[2]].conj(),
                                     basis[node[3]].conj(), basis[i], optimize=True)
    est = float(np.sqrt(max(discarded, 0.0)))
    out = (nodes, frames, transfers)
    return (out, est, eigs) if return_eigs else (out, est)


def dense(h):
    """Dense expansion for tiny cases (reference tests/oracles.py:90-108 pattern)."""
    nodes, frames, transfers = h

    def grow(idx):
        node = nodes[idx]
        if is_leaf(node):
            return frames[idx], node[0]
        left, dl = grow(node[2])
        right, dr = grow(node[3])
        tmp = np.tensordot(left, transfers[idx], axes=(left.ndim - 1, 0))
        out = np.tensordot(tmp, right, axes=(left.ndim - 1, right.ndim - 1))
        out = np.moveaxis(out, left.ndim - 1, -1)
        return out, dl + dr

    out, dims = grow(0)
    return np.transpose(out[..., 0], np.argsort(dims))
