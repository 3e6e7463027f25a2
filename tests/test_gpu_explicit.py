"""GPU parity of the explicit integrator (explicit.py:85-103) with device truncation,
against the oracle (pinned by tests/golden/explicit.npz).  Per-truncation bar
1e-9 (teacher forcing: the GPU truncation gets the oracle's exact input and
init), final-solution bar 1e-8 (BASELINE north star)."""

import math

import numpy as np
import pytest

from conftest import load_golden, unpack_cp
from oracle import explicit as oex
from oracle import metrics

pytestmark = pytest.mark.gpu

from paper_1803_10270_b200 import cp, explicit, ht, operators, workloads  # noqa: E402
from paper_1803_10270_b200.basis import fourier_diff_matrix  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402


def col_specs(d, q):
    return tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for _ in range(d))


def adv_op(S, D, a):
    d = len(S)
    return operators.SeparableOperator(S, tuple(-np.asarray(a)), tuple(tuple(D if k == t else None for k in range(d))
                                                                      for t in range(d)))


def test_fused_trajectory_golden():
    g = load_golden("explicit")
    q, d, r, dt, steps, sweeps, lam = g["meta"]
    q, d, r, steps, sweeps = int(q), int(d), int(r), int(steps), int(sweeps)
    S = col_specs(d, q)
    L = adv_op(S, g["D"], g["a"])
    cfg = explicit.ExplicitConfig(dt=float(dt), r_max=r, recipe="fused",
                                  als=cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=float(lam)))
    f0 = cp.CPTensor(S, unpack_cp(g, "step0"))
    got = {}
    explicit.run(f0, L, cfg, steps, callback=lambda n, f: got.__setitem__(n, f.to_numpy()))
    for n in range(1, steps + 1):
        rel = metrics.cp_rel_diff(unpack_cp(g, f"step{n}"), got[n])
        assert rel <= 1e-8, (n, rel)
    # same through the per-step API
    f1 = explicit.startup_step(f0, L, cfg)
    assert metrics.cp_rel_diff(unpack_cp(g, "step1"), f1.to_numpy()) <= 1e-9
    f2 = explicit.ab2_step(f0, f1, L, cfg)
    assert metrics.cp_rel_diff(unpack_cp(g, "step2"), f2.to_numpy()) <= 1e-8


def _cfg0_setup(steps):
    w = workloads.cfg0(0)
    S = w["specs"]
    L = adv_op(S, w["D"], w["a"])
    cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                  als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
    mats = [[w["D"] if k == t else None for k in range(6)] for t in range(6)]
    return w, S, L, cfg, mats


def test_config0_teacher_forced_truncations():
    w, S, L, cfg, mats = _cfg0_setup(8)
    f0 = w["ic"]["factors"]
    red = oex.warm_als_reducer(w["sweeps"], w["lam"])
    prev, cur = f0, oex.startup_fused(f0, list(-np.asarray(w["a"])), mats, w["dt"], w["r"], red)
    for n in range(2, 8):
        target = oex.ab2_target(prev, cur, list(-np.asarray(w["a"])), mats, w["dt"])
        ref = red(target, cur)
        got = cp.cp_approx_als(cp.CPTensor(S, target), w["r"], cfg.als, init=cp.CPTensor(S, cur))
        rel = metrics.cp_rel_diff(ref, got.to_numpy())
        assert rel <= 1e-9, (n, rel)
        # the device AB2 target matches the oracle's exactly (same column order)
        tgt = explicit.ab2_target(cp.CPTensor(S, prev), cp.CPTensor(S, cur), L, w["dt"])
        assert metrics.cp_rel_diff(target, tgt.to_numpy()) <= 1e-14
        prev, cur = cur, ref


def test_config0_full_trajectory():
    """100 steps of BASELINE config 0; final solution vs oracle <= 1e-8 and vs the
    exact shifted solution within the oracle's own truncation error (+10%)."""
    w, S, L, cfg, mats = _cfg0_setup(100)
    f0 = w["ic"]["factors"]
    out = explicit.run(cp.CPTensor(S, f0), L, cfg, w["steps"])
    ref = oex.run_fused(f0, list(-np.asarray(w["a"])), mats, w["dt"], w["r"], w["steps"], w["sweeps"], w["lam"])
    rel = metrics.cp_rel_diff(ref, out.to_numpy())
    assert rel <= 1e-8, rel
    exact = workloads.advection_exact(w["ic"], w["steps"] * w["dt"])
    e_ref = metrics.cp_rel_diff(exact, ref)
    e_gpu = metrics.cp_rel_diff(exact, out.to_numpy())
    assert e_gpu <= 1.1 * e_ref + 1e-12, (e_gpu, e_ref)
    assert e_ref < 5e-3


def test_config3_short_trajectory():
    w = workloads.cfg3(0)
    S = w["specs"]
    L = operators.SeparableOperator(S, tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
    cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                  als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
    steps = 6
    out = explicit.run(cp.CPTensor(S, w["factors"]), L, cfg, steps)
    ref = oex.run_fused(w["factors"], w["weights"], w["mats"], w["dt"], w["r"], steps, w["sweeps"], w["lam"])
    rel = metrics.cp_rel_diff(ref, out.to_numpy())
    assert rel <= 1e-8, rel


def test_split_recipe_matches_dense_formula_when_untruncated():
    """Rank cap above need: every reduction is a no-op (reference test_explicit.py:35-52)."""
    rng = np.random.default_rng(2)
    d, q = 3, 8
    S = col_specs(d, q)
    D = fourier_diff_matrix(q)
    L = adv_op(S, D, (1.0, 0.5, -0.75))
    f0 = [rng.standard_normal((q, 2)) for _ in range(d)]
    f1 = [rng.standard_normal((q, 2)) for _ in range(d)]
    cfg = explicit.ExplicitConfig(dt=1e-3, r_max=1000)
    out = explicit.ab2_step(cp.CPTensor(S, f0), cp.CPTensor(S, f1), L, cfg)
    mats = [[D if k == t else None for k in range(d)] for t in range(d)]
    ref = oex.ab2_target(f0, f1, [-1.0, -0.5, 0.75], mats, 1e-3)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= 1e-13
    # HT format through the same API
    h0, h1 = ht.from_cp(cp.CPTensor(S, f0)), ht.from_cp(cp.CPTensor(S, f1))
    cfg_ht = explicit.ExplicitConfig(dt=1e-3, r_max=1000, format="ht")
    out_h = explicit.ab2_step(h0, h1, L, cfg_ht)
    from oracle import ht_hsvd as oht
    assert metrics.ht_rel_diff(oht.from_cp(ref), out_h.to_oracle()) <= 1e-12


def test_reduction_log_and_validation():
    rng = np.random.default_rng(4)
    d, q = 3, 8
    S = col_specs(d, q)
    L = adv_op(S, fourier_diff_matrix(q), (1.0, 0.5, -0.75))
    f0 = cp.CPTensor(S, [rng.standard_normal((q, 1)) for _ in range(d)])
    f1 = cp.CPTensor(S, [rng.standard_normal((q, 1)) for _ in range(d)])
    log = []
    out = explicit.ab2_step(f0, f1, L, explicit.ExplicitConfig(dt=1e-3, r_max=2), log=log)
    assert [r.stage for r in log] == ["difference", "operator", "update"]
    assert explicit.tensor_rank(out) <= 2
    assert log[0].rank_before == 2 and log[0].error == 0.0
    assert log[1].rank_before == 6 and log[1].rank_after <= 2
    with pytest.raises(TypeError, match="same tensor format"):
        explicit.ab2_step(f0, ht.from_cp(f1), L, explicit.ExplicitConfig(dt=1e-3, r_max=4))


@pytest.mark.parametrize("which,steps", [("cfg0", 12), ("cfg3", 6)])
def test_graph_replay_matches_eager(which, steps):
    """explicit.run captures one AB2 step in a CUDA graph and replays it: the
    trajectory must be bitwise identical to the eager launches."""
    import torch
    if which == "cfg0":
        w, S, L, cfg, _ = _cfg0_setup(steps)
        f0 = cp.CPTensor(S, w["ic"]["factors"])
    else:
        w = workloads.cfg3(0)
        S = w["specs"]
        L = operators.SeparableOperator(S, tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
        cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                      als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
        f0 = cp.CPTensor(S, w["factors"])
    a = explicit.run(f0, L, cfg, steps, graph=False)
    b = explicit.run(f0, L, cfg, steps, graph=True)
    assert torch.equal(a.data, b.data)


def test_graph_cache_reuse_new_initial_state():
    """The captured AB2 step is cached per operator/configuration; a second run with a
    different initial state must replay on its own data (equal to the eager result)."""
    import torch
    w, S, L, cfg, _ = _cfg0_setup(8)
    f0 = cp.CPTensor(S, w["ic"]["factors"])
    g0 = cp.scale(f0, 0.5)
    a1 = explicit.run(f0, L, cfg, 8, graph=True)
    a2 = explicit.run(g0, L, cfg, 8, graph=True)     # cached graph, new states
    b2 = explicit.run(g0, L, cfg, 8, graph=False)
    b1 = explicit.run(f0, L, cfg, 8, graph=False)
    assert torch.equal(a1.data, b1.data) and torch.equal(a2.data, b2.data)
    assert not torch.equal(a1.data, a2.data)


@pytest.mark.parametrize("graph", [False, True])
def test_fused_apply_truncation_bitwise(graph):
    """with the one-CTA kernel every truncation of explicit.run assembles its
    target [f1 | dt/2 L(3 f1 - f0)] inside the kernel from the states and the operator's
    matrices (tp_cp_als_recipe_f64, L w never materialised); the trajectory is bitwise
    equal to materialising the target with the apply kernel first."""
    import torch
    w, S, L, cfg, _ = _cfg0_setup(10)
    f0 = cp.CPTensor(S, w["ic"]["factors"])
    assert cp.als_plan(f0.qs, f0.rank + L.n_terms * 2 * f0.rank, f0.rank)["kernel"] == "als_tiny8"
    a = explicit.run(f0, L, cfg, 10, graph=graph, fused=True)
    b = explicit.run(f0, L, cfg, 10, graph=graph, fused=False)
    assert torch.equal(a.data, b.data)


def test_fused_apply_entry_matches_materialised():
    """tp_cp_als_recipe_f64 directly on a random two-block recipe with a mix of identity and
    dense operator factors (incl. several matrices on one mode): bitwise equal to
    cp.concat + operators.apply_into + cp.cp_approx_als."""
    import torch
    rng = np.random.default_rng(5)
    qs, r = (9, 12, 7, 10), 5
    S = tuple(BasisSpec(q, 1.0, "collocation") for q in qs)
    f1 = cp.CPTensor(S, [rng.standard_normal((q, r)) for q in qs])
    f0 = cp.CPTensor(S, [rng.standard_normal((q, r)) for q in qs])
    mats = [[rng.standard_normal((q, q)) / q if (t + k) % 3 == 0 else None for k, q in enumerate(qs)]
            for t in range(5)]
    L = operators.SeparableOperator(S, tuple(rng.uniform(-1, 1, 5)), tuple(tuple(m) for m in mats))
    acfg = cp.ALSApproxConfig(max_sweeps=7, stall=-np.inf, reg=1e-10)
    info = torch.zeros(2, dtype=torch.int32, device=f1.data.device)
    U = explicit._fused_trunc(f1, [(f1, 3.0), (f0, -1.0)], L, 0.05, f1, r, acfg, info)
    assert U is not None
    tgt = explicit.ab2_target(f0, f1, L, 0.1)
    ref = cp.cp_approx_als(tgt, r, acfg, init=f1)
    assert int(info[0]) == 0
    assert torch.equal(U, ref.data)
