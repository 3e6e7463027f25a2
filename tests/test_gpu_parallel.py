"""GPU parity of the R-sharded ALS mode-step kernels (tp_als_shard_*).  N shards
are simulated on one GPU in lockstep: every shard computes its right-hand-side
partial, the host sums them (the allreduce), every shard finishes the mode.  No
kernel waits on another, so this is safe on a single device; the multi-process
orchestration itself is covered by tests/test_parallel.py (gloo)."""

import math

import numpy as np
import pytest
import torch

from oracle import cp_als as ocp
from oracle import metrics

pytestmark = pytest.mark.gpu

from paper_1803_10270_b200 import cp, parallel, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402


def run_simulated(V, init, world, sweeps, lam=1e-10):
    qs = [v.shape[0] for v in V]
    S = tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for q in qs)
    R, r = V[0].shape[1], init[0].shape[1]
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=lam)
    shards = []
    for g in range(world):
        lo, hi = parallel.shard_range(R, world, g)
        Vs = cp.CPTensor(S, [v[:, lo:hi] for v in V])
        U = cp.CPTensor(S, init).data
        drv = parallel.ShardedALS(parallel.DeviceShardOps(Vs, r), parallel.LocalComm(), cfg)
        drv.begin(U)
        shards.append(drv)
    for _ in range(sweeps):
        for j in range(len(V)):
            parts = [s.mode_rhs(j) for s in shards]
            tot = parts[0].clone()
            for p in parts[1:]:
                tot += p
            for s in shards:
                s.mode_finish(j, tot)
    outs = []
    for s in shards:
        s.ops.check()
        u = s.U.cpu().numpy()
        fac, off = [], 0
        for q in qs:
            fac.append(u[off:off + q * r].reshape(q, r))
            off += q * r
        outs.append(fac)
    return outs


@pytest.mark.parametrize("world", [1, 2, 4, 7])
def test_simulated_shards_match_oracle(world):
    rng = np.random.default_rng(3)
    qs, R, r, sweeps = (20, 16, 24, 12), 41, 6, 8
    V = [rng.standard_normal((q, R)) / 4 for q in qs]
    init = [v[:, :r].copy() for v in V]
    outs = run_simulated(V, init, world, sweeps)
    ref = ocp.als(V, init, sweeps, lam=1e-10)
    for o in outs:
        assert metrics.cp_rel_diff(ref, o) <= 1e-9
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            np.testing.assert_array_equal(a, b)


def test_config1_two_shards_full_size():
    w = workloads.cfg1(seed=0)
    outs = run_simulated(w["V"], w["init"], 2, w["sweeps"], w["lam"])
    ref = ocp.als(w["V"], w["init"], w["sweeps"], lam=w["lam"])
    assert metrics.cp_rel_diff(ref, outs[0]) <= 1e-9


def test_sharded_api_single_rank_equals_fused_kernel():
    rng = np.random.default_rng(4)
    qs, R, r = (16, 16, 16, 16), 30, 8
    S = tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for q in qs)
    V = [rng.standard_normal((q, R)) / 4 for q in qs]
    init = cp.CPTensor(S, [v[:, :r].copy() for v in V])
    cfg = cp.ALSApproxConfig(max_sweeps=10, stall=-np.inf, reg=1e-10)
    a = parallel.sharded_cp_approx_als(cp.CPTensor(S, V), init, cfg)
    b = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=init)
    assert metrics.cp_rel_diff(b.to_numpy(), a.to_numpy()) <= 1e-12
    _ = torch


def test_captured_graph_replay_matches_eager():
    rng = np.random.default_rng(5)
    qs, R, r = (16, 12, 20), 25, 5
    S = tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for q in qs)
    V = [rng.standard_normal((q, R)) / 4 for q in qs]
    init = cp.CPTensor(S, [v[:, :r].copy() for v in V])
    cfg = cp.ALSApproxConfig(max_sweeps=7, stall=-np.inf, reg=1e-10)
    ops = parallel.DeviceShardOps(cp.CPTensor(S, V), r)
    drv = parallel.ShardedALS(ops, parallel.LocalComm(), cfg)
    U = init.data.clone()
    drv.capture(U, len(qs))
    U.copy_(init.data)
    drv.replay()
    torch.cuda.synchronize()
    ref = ocp.als(V, [v[:, :r].copy() for v in V], 7, lam=1e-10)
    out = cp.CPTensor(S, data=U, rank=r).to_numpy()
    assert metrics.cp_rel_diff(ref, out) <= 1e-9
