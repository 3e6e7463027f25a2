"""Single-file tensor format of the reference (mirror of ``tensorpde/io.py``).

One UTF-8 JSON header line, then little-endian complex128 coefficients
(io.py:1-10).  CP tensors: ``{format: "cp", version: 1, N, r, Q, b}`` with the
payload term-major, dimension middle, mode minor (io.py:28-36, 58-59); HT tensors:
``{format: "ht", ...}`` with the tree as parallel dims/parent/left/right arrays and
the per-node ranks, payload = every node's array (leaf frame Q x k, interior
transfer k_l x k_r x k) in node order, C order (io.py:39-52, 60-63, 95-112).

Real-valued tensors are stored in real fp64 on the device and written with zero
imaginary parts; files are byte-identical to the reference's for Fourier-basis
specs (the header gains ``kind``/``lo`` keys only for the build's collocation /
uniform grids).  A CP file with non-zero imaginary parts loads as a complex128
CPTensor (the reference's own arithmetic); an HT file with
non-zero imaginary parts raises ``ValueError`` (the hSVD path is real fp64).  The pure ``encode_*`` / ``decode``
functions work on numpy arrays; ``save_tensor`` / ``load_tensor`` move the
device tensors.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .basis import BasisSpec

__all__ = ["save_tensor", "load_tensor", "encode_cp", "encode_ht", "decode"]

_DTYPE = np.dtype("<c16")


def _spec_header(specs) -> dict:
    h = {"Q": [int(s.Q) for s in specs], "b": [float(s.b) for s in specs]}
    if any(s.kind != "fourier" for s in specs):
        h["kind"] = [s.kind for s in specs]
        h["lo"] = [s.lo for s in specs]
    return h


def _specs_from(header) -> tuple:
    kinds = header.get("kind") or ["fourier"] * len(header["Q"])
    los = header.get("lo") or [None] * len(header["Q"])
    return tuple(BasisSpec(int(q), float(b), k, lo) for q, b, k, lo in zip(header["Q"], header["b"], kinds, los))


def _pack(header: dict, blocks) -> bytes:
    payload = (np.concatenate([np.ascontiguousarray(b, dtype=complex).reshape(-1) for b in blocks])
               if blocks else np.zeros(0, dtype=complex)).astype(_DTYPE)
    return json.dumps(header).encode() + b"\n" + payload.tobytes()


def encode_cp(specs, factors) -> bytes:
    """io.py:28-36 header, io.py:58-59 payload (term l, then dimension k, column of Q_k)."""
    factors = [np.asarray(f) for f in factors]
    r = int(factors[0].shape[1])
    header = {"format": "cp", "version": 1, "N": len(specs), "r": r}
    header.update(_spec_header(specs))
    return _pack(header, [factors[k][:, l] for l in range(r) for k in range(len(specs))])


def encode_ht(specs, nodes, frames, transfers, ranks) -> bytes:
    """io.py:39-52 header, io.py:60-63 payload.  ``nodes``: (dims, parent, left, right)."""
    header = {"format": "ht", "version": 1, "N": len(specs)}
    header.update(_spec_header(specs))
    header.update({"dims": [list(n[0]) for n in nodes], "parent": [int(n[1]) for n in nodes],
                   "left": [int(n[2]) for n in nodes], "right": [int(n[3]) for n in nodes],
                   "ranks": [int(x) for x in ranks]})
    blocks = [np.asarray(frames[i] if n[2] < 0 else transfers[i]).reshape(-1) for i, n in enumerate(nodes)]
    return _pack(header, blocks)


def decode(raw: bytes):
    """io.py:74-115.  Returns ("cp", specs, factors) or ("ht", specs, nodes, frames, transfers),
    numpy complex arrays."""
    cut = raw.index(b"\n")
    header = json.loads(raw[:cut].decode())
    payload = np.frombuffer(raw[cut + 1:], dtype=_DTYPE).astype(complex)
    fmt = header.get("format")
    if fmt not in ("cp", "ht"):
        raise ValueError(f"unknown tensor format {fmt!r}")
    specs = _specs_from(header)
    if fmt == "cp":
        n, r = header["N"], header["r"]
        if payload.size != r * sum(s.Q for s in specs):
            raise ValueError("payload length does not match the header")
        factors = [np.empty((s.Q, r), dtype=complex) for s in specs]
        pos = 0
        for l in range(r):
            for k in range(n):
                q = specs[k].Q
                factors[k][:, l] = payload[pos:pos + q]
                pos += q
        return "cp", specs, factors
    nodes = [(tuple(d), p, lf, rt) for d, p, lf, rt in zip(header["dims"], header["parent"], header["left"],
                                                            header["right"])]
    ranks = header["ranks"]
    frames, transfers = [None] * len(nodes), [None] * len(nodes)
    pos = 0
    for i, (dims, _, left, right) in enumerate(nodes):
        shape = (specs[dims[0]].Q, ranks[i]) if left < 0 else (ranks[left], ranks[right], ranks[i])
        size = int(np.prod(shape))
        if pos + size > payload.size:
            raise ValueError("payload length does not match the header")
        block = payload[pos:pos + size].reshape(shape)
        pos += size
        if left < 0:
            frames[i] = block
        else:
            transfers[i] = block
    if pos != payload.size:
        raise ValueError("payload length does not match the header")
    return "ht", specs, nodes, frames, transfers


def save_tensor(path, t) -> None:
    """io.py:55-71 for the device CPTensor / HTTensor."""
    from .cp import CPTensor
    from .ht import HTTensor
    if isinstance(t, CPTensor):
        raw = encode_cp(t.specs, t.to_numpy())
    elif isinstance(t, HTTensor):
        nodes, frames, transfers = t.to_oracle()
        raw = encode_ht(t.specs, nodes, frames, transfers, t.ranks)
    else:
        raise TypeError(f"cannot serialize {type(t).__name__}")
    Path(path).write_bytes(raw)


def load_tensor(path):
    """io.py:74-115 -> device CPTensor (real fp64, or complex128 when the payload has
    non-zero imaginary parts) / HTTensor (real fp64; complex payloads raise)."""
    from .cp import CPTensor
    from .ht import DimensionTree, HTTensor, TreeNode
    out = decode(Path(path).read_bytes())
    if out[0] == "cp":
        _, specs, factors = out
        return CPTensor(specs, factors)
    _, specs, nodes, frames, transfers = out
    tree = DimensionTree(tuple(TreeNode(tuple(d), p, lf, rt) for d, p, lf, rt in nodes))
    return HTTensor(specs, tree, frames, transfers)
