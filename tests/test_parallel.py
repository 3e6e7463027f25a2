"""Multi-rank host logic of the R-sharded ALS with world_size 2 over
gloo on CPU, plus the config-4 batch split.  The per-shard arithmetic here is a
test-only numpy implementation of the DeviceShardOps interface (the product
kernels are covered by the GPU tests in test_gpu_parallel.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cp_als as ocp
from oracle import metrics
from paper_1803_10270_b200 import parallel
from paper_1803_10270_b200.cp import ALSApproxConfig


class NumpyShardOps:
    """Reference arithmetic of one shard (cp.py:190-203, 312-320) -- test only."""

    def __init__(self, V_slab, r):
        self.V, self.r = [np.asarray(v) for v in V_slab], r

    def init(self, U):
        self.Uv = U  # torch CPU tensor (flat CP layout)
        u = self._u()
        self.C = [uk.T @ vk for uk, vk in zip(u, self.V)]
        self.G = [uk.T @ uk for uk in u]

    def _u(self):
        out, off = [], 0
        for v in self.V:
            n = v.shape[0] * self.r
            out.append(self.Uv[off:off + n].view(v.shape[0], self.r).numpy())
            off += n
        return out

    def rhs(self, j):
        had = np.ones_like(self.C[0])
        for k, c in enumerate(self.C):
            if k != j:
                had = had * c
        return torch.as_tensor(had @ self.V[j].T)

    def update(self, U, j, rhs, reg, reg_mode):
        gram = np.ones((self.r, self.r))
        for k, g in enumerate(self.G):
            if k != j:
                gram = gram * g
        x = np.linalg.solve(gram + reg * np.eye(self.r), rhs.numpy())
        u = self._u()
        u[j][:] = x.T
        self.G[j] = u[j].T @ u[j]
        self.C[j] = u[j].T @ self.V[j]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, V, init, sweeps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R = V[0].shape[1]
    lo, hi = parallel.shard_range(R, world, rank)
    ops = NumpyShardOps([v[:, lo:hi] for v in V], init[0].shape[1])
    U = torch.as_tensor(np.concatenate([u.ravel() for u in init]))
    cfg = ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10)
    parallel.ShardedALS(ops, parallel.TorchDistComm(), cfg).run(U, len(V))
    out_q.put((rank, U.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_als_gloo_matches_unsharded(world):
    rng = np.random.default_rng(1)
    qs, R, r, sweeps = (12, 10, 9), 23, 4, 6
    V = [rng.standard_normal((q, R)) / 3 for q in qs]
    init = [v[:, :r].copy() for v in V]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, world, port, V, init, sweeps, q)) for i in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    ref = ocp.als(V, init, sweeps, lam=1e-10)
    for rank in range(world):
        flat = res[rank]
        out, off = [], 0
        for qq in qs:
            out.append(flat[off:off + qq * r].reshape(qq, r))
            off += qq * r
        assert metrics.cp_rel_diff(ref, out) <= 1e-11
    # every rank holds the identical replicated fit
    for rank in range(1, world):
        np.testing.assert_array_equal(res[0], res[rank])


def test_shard_partitions_cover_exactly():
    for n in (1, 7, 64, 512):
        for world in (1, 2, 3, 8):
            spans = [parallel.shard_range(n, world, g) for g in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    items = list(range(64))
    assert sum((parallel.shard_batch(items, 8, g) for g in range(8)), []) == items
