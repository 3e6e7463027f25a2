"""Full-length final-solution parity of every BASELINE trajectory (north-star gate
<= 1e-8 on final solutions), each reported beside the problem's own sensitivity
at the SAME length (oracle vs the oracle started from a 1e-13 relative
perturbation, tests/golden/make_final_states.py):

* config 0: all 100 fused-AB2 steps (explicit.run, CUDA-graph replay);
* config 3: all 200 fused-AB2 steps;
* config 2: all 50 implicit-Euler steps (20 Gauss-Seidel sweeps each);
* config 4: all 64 tensors of the batch through the public ht.truncate_batch
  (the oracle runs live on the host cores).

Set TPDE_PARITY_LOG=<file> to append one line per config (profiles/)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ht_hsvd as oht
from oracle import metrics

pytestmark = pytest.mark.gpu

from paper_1803_10270_b200 import cp, explicit, ht, implicit, operators, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402


def load(part):
    z = np.load(GOLDEN / f"final_{part}.npz")
    return [z[f"f_{k}"] for k in range(int(z["d"]))]


def log(line):
    path = os.environ.get("TPDE_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(line + "\n")


def _explicit_cfg(w):
    return explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                   als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))


def test_config0_final_100_steps():
    w = workloads.cfg0(0)
    S, d = w["specs"], 6
    L = operators.SeparableOperator(S, tuple(-np.asarray(w["a"])),
                                    tuple(tuple(w["D"] if k == t else None for k in range(d)) for t in range(d)))
    out = explicit.run(cp.CPTensor(S, w["ic"]["factors"]), L, _explicit_cfg(w), w["steps"]).to_numpy()
    ref, pert = load("cfg0"), load("cfg0p")
    rel, sens = metrics.cp_rel_diff(ref, out), metrics.cp_rel_diff(ref, pert)
    log(f"cfg0 final after 100 steps: gpu vs oracle {rel:.2e}; oracle vs 1e-13-perturbed oracle {sens:.2e}")
    assert rel <= 1e-8, rel


def test_config3_final_200_steps():
    w = workloads.cfg3(0)
    S = w["specs"]
    L = operators.SeparableOperator(S, tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
    out = explicit.run(cp.CPTensor(S, w["factors"]), L, _explicit_cfg(w), w["steps"]).to_numpy()
    ref, pert = load("cfg3"), load("cfg3p")
    rel, sens = metrics.cp_rel_diff(ref, out), metrics.cp_rel_diff(ref, pert)
    log(f"cfg3 final after 200 steps: gpu vs oracle {rel:.2e}; oracle vs 1e-13-perturbed oracle {sens:.2e}")
    assert rel <= 1e-8, rel


@pytest.mark.parametrize("solver", ["circulant", "dense"])
def test_config2_final_50_steps(solver):
    w = workloads.cfg2(0)
    S, D, a, dt = w["specs"], w["D"], w["a"], w["dt"]
    pair = operators.implicit_euler_pair(operators.advection_operator(a, S), dt)
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=w["sweeps"], delta_beta=1.0,
                                 schedule="gauss-seidel", lam=w["lam"], solver=solver)
    out = implicit.run(cp.CPTensor(S, w["ic"]["factors"]), pair, cfg, w["steps"]).to_numpy()
    ref, pert = load("cfg2"), load("cfg2p")
    rel, sens = metrics.cp_rel_diff(ref, out), metrics.cp_rel_diff(ref, pert)
    log(f"cfg2 ({solver}) final after 50 steps: gpu vs oracle {rel:.2e}; "
        f"oracle vs 1e-13-perturbed oracle {sens:.2e}")
    assert rel <= 1e-8, rel


def _cfg4_oracle_tensor(w, b):
    nodes = oht.balanced_tree(w["d"])
    frames, transfers, li, ii = [None] * len(nodes), [None] * len(nodes), 0, 0
    for t, nd in enumerate(nodes):
        if oht.is_leaf(nd):
            frames[t] = w["frames"][b, li]
            li += 1
        else:
            transfers[t] = w["transfers"][b, ii][:, :, :1] if t == 0 else w["transfers"][b, ii]
            ii += 1
    return nodes, frames, transfers


def test_config4_full_batch_64():
    w = workloads.cfg4(0)
    d, Q = w["d"], w["Q"]
    specs = tuple(BasisSpec(Q, 1.0, "collocation") for _ in range(d))
    hs = []
    for b in range(64):
        _, frames, transfers = _cfg4_oracle_tensor(w, b)
        hs.append(ht.HTTensor(specs, ht.balanced_tree(d), frames, transfers))
    outs, ests = ht.truncate_batch(hs, w["r_max"], w["eps"])
    worst, worst_est = 0.0, 0.0
    for b in range(64):
        o = _cfg4_oracle_tensor(w, b)
        ref, oest = oht.truncate(o, w["r_max"], w["eps"])
        rel = metrics.ht_rel_diff(ref, outs[b].to_oracle())
        worst = max(worst, rel)
        worst_est = max(worst_est, abs(ests[b] - oest) / oht.norm(o))
        assert outs[b].max_rank == 16
    log(f"cfg4 all 64 tensors: worst gpu vs oracle {worst:.2e}; worst |est - oracle est|/|h| {worst_est:.2e}")
    assert worst <= 1e-9, worst
    assert worst_est <= 1e-9, worst_est
