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


# ---- fused one-launch R-sharded kernel (tp_als_xg_f64) ------------------------------

def _unflat(u, qs, r):
    u = u.cpu().numpy()
    fac, off = [], 0
    for q in qs:
        fac.append(u[off:off + q * r].reshape(q, r))
        off += q * r
    return fac


@pytest.mark.parametrize("shards", [1, 2, 4])
@pytest.mark.parametrize("qs,R,r", [((20, 16, 24, 12), 48, 6), ((32, 40, 28), 64, 16), ((64,) * 4, 96, 32)])
def test_fused_sharded_simulated_groups(shards, qs, R, r):
    """`shards` ranks' CTA groups in ONE launch (the in-kernel peer exchange and
    cross-group flag barrier exactly as across GPUs): every rank's fit is bitwise
    identical and matches the oracle (cp.py:310-320) at <= 1e-9."""
    rng = np.random.default_rng(R + r + shards)
    V = [rng.standard_normal((q, R)) / 4 for q in qs]
    init = [v[:, :r].copy() for v in V]
    sweeps = 7
    outs = parallel.simulate_sharded_als(V, init, shards, cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf,
                                                                              reg=1e-10))
    for u in outs[1:]:
        assert torch.equal(u, outs[0])
    ref = ocp.als(V, init, sweeps, lam=1e-10)
    assert metrics.cp_rel_diff(ref, _unflat(outs[0], qs, r)) <= 1e-9


@pytest.mark.parametrize("shards", [2, 4])
def test_fused_sharded_config1(shards):
    """BASELINE config 1 (d=6, Q=256, R=512 -> r=32, 20 sweeps) R-sharded over 2 / 4
    simulated ranks: bitwise-identical replicas, oracle parity <= 1e-9."""
    w = workloads.cfg1(seed=1)
    outs = parallel.simulate_sharded_als(w["V"], w["init"], shards,
                                         cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
    for u in outs[1:]:
        assert torch.equal(u, outs[0])
    ref = ocp.als(w["V"], w["init"], w["sweeps"], lam=w["lam"])
    assert metrics.cp_rel_diff(ref, _unflat(outs[0], [256] * 6, 32)) <= 1e-9


def test_fused_sharded_driver_world1_repeatable():
    """FusedShardedALS on one rank (no process group): the public sharded API, repeated
    calls (monotonic barrier tags across launches) give identical fits, oracle parity."""
    rng = np.random.default_rng(8)
    qs, R, r = (48, 40, 36, 44), 80, 12
    S = tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for q in qs)
    V = [rng.standard_normal((q, R)) / 4 for q in qs]
    init = [v[:, :r].copy() for v in V]
    cfg = cp.ALSApproxConfig(max_sweeps=6, stall=-np.inf, reg=1e-10)
    Vt, It = cp.CPTensor(S, V), cp.CPTensor(S, init)
    outs = [parallel.sharded_cp_approx_als(Vt, It, cfg) for _ in range(3)]
    for o in outs[1:]:
        assert torch.equal(o.data, outs[0].data)
    ref = ocp.als(V, init, 6, lam=1e-10)
    assert metrics.cp_rel_diff(ref, outs[0].to_numpy()) <= 1e-9
    drv = parallel.make_sharded_als(Vt, r, cfg)
    assert isinstance(drv, parallel.FusedShardedALS)
    U = It.data.clone()
    drv.run(U)
    drv.check()
    assert torch.equal(U, outs[0].data)
    drv.close()
