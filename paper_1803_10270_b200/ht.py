"""Hierarchical Tucker tensors on the device and hSVD truncation (mirror of
``tensorpde/ht.py``).

Frames (leaf bases, ``(Q_k, r_i)``) and transfer tensors (``(r_left, r_right,
r_node)``, root rank 1) are fp64 device tensors indexed by tree node exactly as
in the reference (ht.py:101-157).  ``truncate`` and ``truncate_batch`` run the
batched sm_100a hSVD kernels of ``tp_ht_truncate_f64``; ragged ranks / mode
sizes are zero-padded to a uniform batch layout on the device (exact: zero
columns add zero eigenvalues, which the keep rule drops).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cp import CPTensor

__all__ = ["TreeNode", "DimensionTree", "balanced_tree", "HTTensor", "from_cp", "add", "scale",
           "inner_product", "norm", "truncate", "truncate_batch", "apply_operator", "HTBatch", "truncate_packed"]


@dataclass(frozen=True)
class TreeNode:
    dims: tuple
    parent: int
    left: int
    right: int

    @property
    def is_leaf(self) -> bool:
        return self.left < 0


@dataclass(frozen=True)
class DimensionTree:
    """ht.py:55-76: nodes[0] is the root, preorder indices."""

    nodes: tuple

    def __post_init__(self):
        if not self.nodes or self.nodes[0].parent != -1:
            raise ValueError("nodes[0] must be the root")
        seen = sorted(d for n in self.nodes if n.is_leaf for d in n.dims)
        if seen != list(range(len(seen))):
            raise ValueError("leaves must partition the dimensions")

    @property
    def ndim(self) -> int:
        return len(self.nodes[0].dims)

    @property
    def leaf_of(self) -> dict:
        return {n.dims[0]: i for i, n in enumerate(self.nodes) if n.is_leaf}


def balanced_tree(ndim: int) -> DimensionTree:
    """ht.py:79-98 (left child takes the floor); the C ABI builds the same tree."""
    if ndim < 1:
        raise ValueError("need at least one dimension")
    nodes: list = []

    def build(dims, parent):
        idx = len(nodes)
        nodes.append(None)
        if len(dims) == 1:
            nodes[idx] = TreeNode(dims, parent, -1, -1)
        else:
            half = len(dims) // 2
            left = build(dims[:half], idx)
            right = build(dims[half:], idx)
            nodes[idx] = TreeNode(dims, parent, left, right)
        return idx

    build(tuple(range(ndim)), -1)
    return DimensionTree(tuple(nodes))


def _dev_tensor(x, dev):
    if isinstance(x, torch.Tensor):
        if x.is_complex():
            if torch.any(x.imag != 0):
                raise ValueError("complex coefficients are not supported on the real-fp64 B200 path")
            x = x.real
        return x.detach().to(device=dev, dtype=torch.float64).contiguous()
    a = np.asarray(x)
    if np.iscomplexobj(a):
        if np.any(a.imag != 0):
            raise ValueError("complex coefficients are not supported on the real-fp64 B200 path")
        a = a.real
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


class HTTensor:
    """``frames[i]`` set exactly on leaves, ``transfers[i]`` exactly on interior
    nodes (ht.py:103-134 validation and rank bookkeeping)."""

    def __init__(self, specs, tree: DimensionTree, frames, transfers):
        self.specs = tuple(specs)
        self.tree = tree
        if tree.ndim != len(self.specs):
            raise ValueError("tree does not cover the specs")
        dev = _lib.device()
        frames = list(frames)
        transfers = list(transfers)
        ranks = [0] * len(tree.nodes)
        for i, node in enumerate(tree.nodes):
            if node.is_leaf:
                u = _dev_tensor(frames[i], dev)
                if u.dim() != 2 or u.shape[0] != self.specs[node.dims[0]].Q:
                    raise ValueError(f"bad frame shape at node {i}: {tuple(u.shape)}")
                frames[i] = u
                ranks[i] = u.shape[1]
        for i in reversed(range(len(tree.nodes))):
            node = tree.nodes[i]
            if node.is_leaf:
                continue
            b = _dev_tensor(transfers[i], dev)
            if b.dim() != 3 or tuple(b.shape[:2]) != (ranks[node.left], ranks[node.right]):
                raise ValueError(f"bad transfer shape at node {i}: {tuple(b.shape)}")
            transfers[i] = b
            ranks[i] = b.shape[2]
        if ranks[0] != 1:
            raise ValueError("root rank must be 1")
        self.frames = frames
        self.transfers = transfers
        self._ranks = tuple(ranks)

    @property
    def ndim(self) -> int:
        return len(self.specs)

    @property
    def ranks(self) -> tuple:
        return self._ranks

    @property
    def max_rank(self) -> int:
        return max(self._ranks[1:]) if len(self._ranks) > 1 else 1

    def copy(self) -> "HTTensor":
        return HTTensor(self.specs, self.tree, [None if u is None else u.clone() for u in self.frames],
                        [None if b is None else b.clone() for b in self.transfers])

    def norm(self) -> float:
        return norm(self)

    def to_oracle(self):
        """(nodes, frames, transfers) of numpy arrays in the oracle's tuple format."""
        nodes = [(n.dims, n.parent, n.left, n.right) for n in self.tree.nodes]
        return (nodes, [None if u is None else u.cpu().numpy() for u in self.frames],
                [None if b is None else b.cpu().numpy() for b in self.transfers])


def _check_compatible(h1: HTTensor, h2: HTTensor) -> None:
    if h1.specs != h2.specs or h1.tree != h2.tree:
        raise ValueError("operands live on different trees or domains")


def from_cp(f: CPTensor, tree: DimensionTree | None = None) -> HTTensor:
    """ht.py:165-186: exact conversion, diagonal transfers."""
    tree = tree or balanced_tree(f.ndim)
    r = f.rank
    dev = f.data.device
    frames = [None] * len(tree.nodes)
    transfers = [None] * len(tree.nodes)
    fac = f.factors
    if f.ndim == 1:
        frames[0] = fac[0].sum(dim=1, keepdim=True)
        return HTTensor(f.specs, tree, frames, transfers)
    ar = torch.arange(r, device=dev)
    for i, node in enumerate(tree.nodes):
        if node.is_leaf:
            frames[i] = fac[node.dims[0]].clone()
        elif i == 0:
            root = torch.zeros((r, r, 1), dtype=torch.float64, device=dev)
            root[ar, ar, 0] = 1.0
            transfers[i] = root
        else:
            diag = torch.zeros((r, r, r), dtype=torch.float64, device=dev)
            diag[ar, ar, ar] = 1.0
            transfers[i] = diag
    return HTTensor(f.specs, tree, frames, transfers)


def add(h1: HTTensor, h2: HTTensor) -> HTTensor:
    """ht.py:208-232: block-diagonal concatenation; the root keeps rank 1."""
    _check_compatible(h1, h2)
    frames = [None] * len(h1.tree.nodes)
    transfers = [None] * len(h1.tree.nodes)
    if h1.ndim == 1:
        frames[0] = h1.frames[0] + h2.frames[0]
        return HTTensor(h1.specs, h1.tree, frames, transfers)
    for i, node in enumerate(h1.tree.nodes):
        if node.is_leaf:
            frames[i] = torch.cat([h1.frames[i], h2.frames[i]], dim=1)
            continue
        a, b = h1.transfers[i], h2.transfers[i]
        if i == 0:
            blk = a.new_zeros((a.shape[0] + b.shape[0], a.shape[1] + b.shape[1], 1))
            blk[:a.shape[0], :a.shape[1], 0] = a[:, :, 0]
            blk[a.shape[0]:, a.shape[1]:, 0] = b[:, :, 0]
        else:
            blk = a.new_zeros((a.shape[0] + b.shape[0], a.shape[1] + b.shape[1], a.shape[2] + b.shape[2]))
            blk[:a.shape[0], :a.shape[1], :a.shape[2]] = a
            blk[a.shape[0]:, a.shape[1]:, a.shape[2]:] = b
        transfers[i] = blk
    return HTTensor(h1.specs, h1.tree, frames, transfers)


def scale(h: HTTensor, c) -> HTTensor:
    """ht.py:235-241: scalar folded into the root."""
    c = complex(c)
    if c.imag != 0:
        raise ValueError("complex scalars are not supported on the real-fp64 B200 path")
    out = h.copy()
    if out.tree.nodes[0].is_leaf:
        out.frames[0] = out.frames[0] * c.real
    else:
        out.transfers[0] = out.transfers[0] * c.real
    return out


# ---------------------------------------------------------------------------
# batched device layout

def _pack_batch(hs):
    """Zero-pad a list of HT tensors (same tree/specs) into the uniform batched
    layout of the C ABI: frames (nb, n_leaves, Q, k), transfers (nb, n_int, k, k, k)."""
    h0 = hs[0]
    tree = h0.tree
    dev = h0.frames[[i for i, n in enumerate(tree.nodes) if n.is_leaf][0]].device
    Q = max(s.Q for s in h0.specs)
    k = max(max(h.ranks[1:]) for h in hs)
    leaves = [i for i, n in enumerate(tree.nodes) if n.is_leaf]
    ints = [i for i, n in enumerate(tree.nodes) if not n.is_leaf]
    nb = len(hs)
    F = torch.zeros((nb, len(leaves), Q, k), dtype=torch.float64, device=dev)
    B = torch.zeros((nb, len(ints), k, k, k), dtype=torch.float64, device=dev)
    for b, h in enumerate(hs):
        for s, i in enumerate(leaves):
            u = h.frames[i]
            F[b, s, :u.shape[0], :u.shape[1]] = u
        for s, i in enumerate(ints):
            t = h.transfers[i]
            if i == 0:
                # root (k x k x 1) stored in the first k*k entries of its k^3 slot
                flat = B[b, s].view(-1)[:k * k].view(k, k)
                flat[:t.shape[0], :t.shape[1]] = t[:, :, 0]
            else:
                B[b, s, :t.shape[0], :t.shape[1], :t.shape[2]] = t
    return F, B, Q, k, leaves, ints


def _tree_arrays(tree: DimensionTree):
    n = len(tree.nodes)
    return (n, _lib.int_array([nd.parent for nd in tree.nodes]), _lib.int_array([nd.left for nd in tree.nodes]),
            _lib.int_array([nd.right for nd in tree.nodes]))


def _launch_truncate(tree: DimensionTree, Q, k, nb, F, B, r_max, eps, OF, OB, ranks, est, norms, dev, what):
    """tp_ht_truncate_f64 on balanced trees, tp_ht_truncate_tree_f64 on any other tree."""
    L = _lib.lib()
    d = tree.ndim
    if tree == balanced_tree(d):
        nbytes = L.tp_ht_truncate_ws_bytes(d, Q, k, nb)
        if nbytes == 0:
            raise ValueError(f"unsupported hSVD size d={d}, Q={Q}, k={k}")
        ws = _lib.WORKSPACE.get(nbytes, dev)
        st = L.tp_ht_truncate_f64(d, Q, k, nb, F.data_ptr(), B.data_ptr(), int(r_max), float(eps), OF.data_ptr(),
                                  OB.data_ptr(), ranks.data_ptr(), est.data_ptr(), norms.data_ptr(), ws.data_ptr(),
                                  ws.numel(), _lib.stream_ptr(dev))
    else:
        n, par, lft, rgt = _tree_arrays(tree)
        nbytes = L.tp_ht_truncate_tree_ws_bytes(n, par, lft, rgt, Q, k, nb)
        if nbytes == 0:
            raise ValueError(f"unsupported hSVD size / tree: nodes={n}, Q={Q}, k={k}")
        ws = _lib.WORKSPACE.get(nbytes, dev)
        st = L.tp_ht_truncate_tree_f64(n, par, lft, rgt, Q, k, nb, F.data_ptr(), B.data_ptr(), int(r_max), float(eps),
                                       OF.data_ptr(), OB.data_ptr(), ranks.data_ptr(), est.data_ptr(), norms.data_ptr(),
                                       ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev))
    _lib.check(st, what)


def truncate_batch(hs, r_max: int, eps: float):
    """hSVD-truncate a batch of HT tensors on the same tree in one call.
    Returns (list of HTTensor, list of error estimates)."""
    if r_max < 1:
        raise ValueError("rank cap must be at least 1")
    h0 = hs[0]
    for h in hs[1:]:
        _check_compatible(h0, h)
    tree = h0.tree
    if tree.nodes[0].is_leaf:
        return [h.copy() for h in hs], [0.0] * len(hs)
    F, B, Q, k, leaves, ints = _pack_batch(hs)
    nb = len(hs)
    ro = min(r_max, k)
    dev = F.device
    OF = torch.zeros((nb, len(leaves), Q, ro), dtype=torch.float64, device=dev)
    OB = torch.zeros((nb, len(ints), ro, ro, ro), dtype=torch.float64, device=dev)
    ranks = torch.zeros((nb, len(tree.nodes)), dtype=torch.int32, device=dev)
    est = torch.zeros(nb, dtype=torch.float64, device=dev)
    norms = torch.zeros(nb, dtype=torch.float64, device=dev)
    _launch_truncate(tree, Q, k, nb, F, B, r_max, eps, OF, OB, ranks, est, norms, dev, "truncate")
    ranks_h = ranks.cpu().numpy()
    est_h = est.cpu().numpy()
    outs = []
    for b, h in enumerate(hs):
        rk = ranks_h[b]
        frames = [None] * len(tree.nodes)
        transfers = [None] * len(tree.nodes)
        for s, i in enumerate(leaves):
            frames[i] = OF[b, s, :h.specs[tree.nodes[i].dims[0]].Q, :rk[i]].clone()
        for s, i in enumerate(ints):
            node = tree.nodes[i]
            if i == 0:
                blk = OB[b, s].reshape(-1)[:ro * ro].view(ro, ro)
                transfers[i] = blk[:rk[node.left], :rk[node.right]].unsqueeze(2).clone()
            else:
                transfers[i] = OB[b, s, :rk[node.left], :rk[node.right], :rk[i]].clone()
        outs.append(HTTensor(h.specs, tree, frames, transfers))
    return outs, [float(x) for x in est_h]


class HTBatch:
    """B200 extension of the reference API: ``nb`` HT tensors on one balanced tree,
    held in the packed device layout of ``tp_ht_truncate_f64`` -- frames
    ``(nb, n_leaves, Q, k)`` (leaves in tree order) and transfers
    ``(nb, n_int, k, k, k)`` (interior nodes in tree order, the root's ``k x k x 1``
    in the first ``k*k`` entries of its slot).  ``truncate_packed`` works on it with
    no per-node copies; ``unpack()`` gives the reference-style HTTensor list."""

    def __init__(self, specs, frames: torch.Tensor, transfers: torch.Tensor, ranks=None):
        self.specs = tuple(specs)
        self.tree = balanced_tree(len(self.specs))
        n_leaf = sum(1 for n in self.tree.nodes if n.is_leaf)
        if frames.dim() != 4 or frames.shape[1] != n_leaf or transfers.dim() != 5 \
                or transfers.shape[1] != len(self.tree.nodes) - n_leaf or transfers.shape[0] != frames.shape[0]:
            raise ValueError("packed HT batch layout mismatch")
        if frames.dtype != torch.float64 or transfers.dtype != torch.float64:
            raise ValueError("packed HT batch must be float64")
        if any(s.Q != frames.shape[2] for s in self.specs):
            raise ValueError("packed HT batch needs a uniform mode size Q")
        self.frames, self.transfers = frames, transfers
        k = frames.shape[3]
        self.ranks = ranks if ranks is not None else torch.tensor(
            [[1] + [k] * (len(self.tree.nodes) - 1)] * frames.shape[0], dtype=torch.int32)

    @property
    def nb(self) -> int:
        return self.frames.shape[0]

    @classmethod
    def from_arrays(cls, specs, frames, transfers, non_blocking: bool = False) -> "HTBatch":
        """Upload host arrays (numpy or pinned torch tensors) in two copies."""
        dev = _lib.device()
        f = torch.as_tensor(frames).to(dev, torch.float64, non_blocking=non_blocking)
        t = torch.as_tensor(transfers).to(dev, torch.float64, non_blocking=non_blocking)
        return cls(specs, f, t)

    def unpack(self) -> list:
        tree = self.tree
        leaves = [i for i, n in enumerate(tree.nodes) if n.is_leaf]
        ints = [i for i, n in enumerate(tree.nodes) if not n.is_leaf]
        rk_all = self.ranks.cpu().numpy() if isinstance(self.ranks, torch.Tensor) else np.asarray(self.ranks)
        kk = self.transfers.shape[2]
        outs = []
        for b in range(self.nb):
            rk = rk_all[b]
            frames = [None] * len(tree.nodes)
            transfers = [None] * len(tree.nodes)
            for s, i in enumerate(leaves):
                frames[i] = self.frames[b, s, :, :rk[i]].clone()
            for s, i in enumerate(ints):
                node = tree.nodes[i]
                if i == 0:
                    blk = self.transfers[b, s].reshape(-1)[:kk * kk].view(kk, kk)
                    transfers[i] = blk[:rk[node.left], :rk[node.right]].unsqueeze(2).clone()
                else:
                    transfers[i] = self.transfers[b, s, :rk[node.left], :rk[node.right], :rk[i]].clone()
            outs.append(HTTensor(self.specs, tree, frames, transfers))
        return outs


def truncate_packed(batch: HTBatch, r_max: int, eps: float, out: HTBatch | None = None):
    """hSVD truncation (ht.py:313-372) of a packed batch in one stream-ordered call.
    Returns (HTBatch with ranks <= r_max, zero-padded to min(r_max, k); device tensor
    of error estimates).  No host synchronisation; ``out`` may be reused."""
    if r_max < 1:
        raise ValueError("rank cap must be at least 1")
    d, nb = len(batch.specs), batch.nb
    Q, k = batch.frames.shape[2], batch.frames.shape[3]
    ro = min(r_max, k)
    dev = batch.frames.device
    n_nodes = len(batch.tree.nodes)
    if out is None:
        OF = torch.zeros((nb, d, Q, ro), dtype=torch.float64, device=dev)
        OB = torch.zeros((nb, d - 1, ro, ro, ro), dtype=torch.float64, device=dev)
        out = HTBatch(batch.specs, OF, OB, torch.zeros((nb, n_nodes), dtype=torch.int32, device=dev))
        out.est = torch.zeros(nb, dtype=torch.float64, device=dev)
        out.norms = torch.zeros(nb, dtype=torch.float64, device=dev)
    L = _lib.lib()
    nbytes = L.tp_ht_truncate_ws_bytes(d, Q, k, nb)
    if nbytes == 0:
        raise ValueError(f"unsupported hSVD size d={d}, Q={Q}, k={k}")
    ws = _lib.WORKSPACE.get(nbytes, dev)
    st = L.tp_ht_truncate_f64(d, Q, k, nb, batch.frames.data_ptr(), batch.transfers.data_ptr(), int(r_max),
                              float(eps), out.frames.data_ptr(), out.transfers.data_ptr(), out.ranks.data_ptr(),
                              out.est.data_ptr(), out.norms.data_ptr(), ws.data_ptr(), ws.numel(),
                              _lib.stream_ptr(dev))
    _lib.check(st, "truncate")
    return out, out.est


def truncate(h: HTTensor, r_max: int, eps: float):
    """ht.py:313-372: returns (tensor, sqrt(sum of discarded eigenvalues))."""
    outs, ests = truncate_batch([h], r_max, eps)
    return outs[0], ests[0]


def norm(h: HTTensor) -> float:
    """ht.py:279-282 (computed from the root frame Gram of the hSVD pass)."""
    if h.tree.nodes[0].is_leaf:
        return float(torch.linalg.vector_norm(h.frames[0]).item())
    return float(_norms_batch([h])[0])


def _norms_batch(hs):
    F, B, Q, k, leaves, ints = _pack_batch(hs)
    nb = len(hs)
    dev = F.device
    OF = torch.zeros((nb, len(leaves), Q, 1), dtype=torch.float64, device=dev)
    OB = torch.zeros((nb, len(ints), 1, 1, 1), dtype=torch.float64, device=dev)
    ranks = torch.zeros((nb, len(hs[0].tree.nodes)), dtype=torch.int32, device=dev)
    est = torch.zeros(nb, dtype=torch.float64, device=dev)
    norms = torch.zeros(nb, dtype=torch.float64, device=dev)
    _launch_truncate(hs[0].tree, Q, k, nb, F, B, 1, 0.0, OF, OB, ranks, est, norms, dev, "norm")
    return norms.cpu().numpy()


def inner_product(h1: HTTensor, h2: HTTensor) -> float:
    """ht.py:264-276: leaves-to-root contraction of the two trees on the device.
    Leaf Grams U1^T U2; an interior node folds its children's Grams into its
    transfers, M_t = sum B1[a,b,i] M_l[a,c] M_r[b,d] B2[c,d,j] (two GEMMs and a
    batched one); the root's 1x1 Gram is the inner product (real path)."""
    _check_compatible(h1, h2)
    nodes = h1.tree.nodes
    grams = [None] * len(nodes)
    for i in reversed(range(len(nodes))):
        node = nodes[i]
        if node.is_leaf:
            grams[i] = h1.frames[i].T @ h2.frames[i]
            continue
        b1, b2 = h1.transfers[i], h2.transfers[i]
        ml, mr = grams[node.left], grams[node.right]
        ka, kb, ki = b1.shape
        kc, kd = ml.shape[1], mr.shape[1]
        t = (ml.T @ b1.reshape(ka, kb * ki)).reshape(kc, kb, ki)          # [c, b, i]
        t = (mr.T @ t.permute(1, 0, 2).reshape(kb, kc * ki))               # [d, (c, i)]
        t = t.reshape(kd, kc, ki).permute(1, 0, 2).reshape(kc * kd, ki)   # [(c, d), i]
        grams[i] = t.T @ b2.reshape(kc * kd, b2.shape[2])
    return float(grams[0].reshape(-1)[0].item())


def apply_operator(op, h: HTTensor) -> HTTensor:
    """ht.py:244-261: separable operator acting leaf by leaf, terms summed block-diagonally."""
    from .operators import dense_factor
    if len(op.specs) != h.ndim:
        raise ValueError("operator and tensor dimension mismatch")
    leaf_of = h.tree.leaf_of
    dev = next(u for u in h.frames if u is not None).device
    out = None
    for t in range(op.n_terms):
        frames = list(h.frames)
        for k, m in enumerate(op.factors[t]):
            dm = dense_factor(op.specs[k], m)
            if dm is None:
                continue
            i = leaf_of[k]
            frames[i] = _matmul_dev(torch.as_tensor(dm, device=dev), h.frames[i])
        term = scale(HTTensor(h.specs, h.tree, frames, list(h.transfers)), complex(op.weights[t]))
        out = term if out is None else add(out, term)
    return out


def _matmul_dev(E: torch.Tensor, U: torch.Tensor) -> torch.Tensor:
    """E @ U through the K1 apply kernel (one-mode, one-term apply)."""
    from .basis import BasisSpec
    from .cp import _apply_raw
    q, r = U.shape
    spec = (BasisSpec(q, 1.0, "collocation"),)
    f = CPTensor(spec, data=U.contiguous().view(-1), rank=r)
    out = CPTensor(spec, data=torch.empty(q * r, dtype=torch.float64, device=U.device), rank=r)
    _apply_raw(f, [[0]], [1.0], 1.0, E.contiguous().view(-1), out, 0, [0])
    return out.data.view(q, r)
