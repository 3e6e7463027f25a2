"""Parity beside conditioning, per BASELINE config (SURVEY 8(d) "Measured conditioning"):

  gpu      = rel(oracle(x), gpu(x))                       -- the parity number
  perturb  = rel(oracle(x), oracle(x (1 + 1e-13 xi)))     -- the problem's own amplification of
                                                             a 1e-13 relative input perturbation
rel() is the HT-orthogonalised metric of oracle/metrics.py (never the Gram identity).
Sizes: config 1 one full truncation; config 0 100 steps; config 3 6 steps; config 2 one step
with 3 sweeps; config 4 one tensor.  python tools/sensitivity.py [cfg ...]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import cp_als as ocp  # noqa: E402
from oracle import explicit as oex  # noqa: E402
from oracle import ht_hsvd as oht  # noqa: E402
from oracle import implicit as oim  # noqa: E402
from oracle import metrics  # noqa: E402
from paper_1803_10270_b200 import cp, explicit, ht, implicit, operators, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402

EPS = 1e-13
rng = np.random.default_rng(123)


def perturb(fs):
    return [f * (1.0 + EPS * rng.standard_normal(f.shape)) for f in fs]


def cfg1():
    w = workloads.cfg1(0)
    V, I0 = w["V"], w["init"]
    ref = ocp.als(V, I0, w["sweeps"], lam=w["lam"])
    pert = ocp.als(V, perturb(I0), w["sweeps"], lam=w["lam"])
    out = cp.cp_approx_als(cp.CPTensor(w["specs"], V), 32,
                           cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]),
                           init=cp.CPTensor(w["specs"], I0)).to_numpy()
    return metrics.cp_rel_diff(ref, out), metrics.cp_rel_diff(ref, pert), "one 20-sweep truncation (init perturbed)"


def _explicit(w, weights, mats, L, f0, steps):
    cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                  als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
    ref = oex.run_fused(f0, weights, mats, w["dt"], w["r"], steps, w["sweeps"], w["lam"])
    pert = oex.run_fused(perturb(f0), weights, mats, w["dt"], w["r"], steps, w["sweeps"], w["lam"])
    out = explicit.run(cp.CPTensor(w["specs"], f0), L, cfg, steps).to_numpy()
    return metrics.cp_rel_diff(ref, out), metrics.cp_rel_diff(ref, pert)


def cfg0():
    w = workloads.cfg0(0)
    d = len(w["specs"])
    a = list(-np.asarray(w["a"]))
    mats = [[w["D"] if k == t else None for k in range(d)] for t in range(d)]
    L = operators.SeparableOperator(w["specs"], tuple(a), tuple(tuple(m) for m in mats))
    g, p = _explicit(w, a, mats, L, w["ic"]["factors"], w["steps"])
    return g, p, "100 fused-AB2 steps (initial condition perturbed)"


def cfg3():
    w = workloads.cfg3(0)
    L = operators.SeparableOperator(w["specs"], tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
    g, p = _explicit(w, w["weights"], w["mats"], L, w["factors"], 6)
    return g, p, "6 fused-AB2 steps (initial condition perturbed)"


def cfg2():
    w = workloads.cfg2(0)
    S, D, a, dt = w["specs"], w["D"], w["a"], w["dt"]
    d, q = len(S), S[0].Q
    f0 = w["ic"]["factors"]
    sweeps = 3
    mats = [[D if k == t else None for k in range(d)] for t in range(d)]
    L = operators.SeparableOperator(S, tuple(-np.asarray(a)), tuple(tuple(m) for m in mats))
    pair = operators.implicit_euler_pair(L, dt)
    eta = [1.0] + [dt * x for x in a]
    zeta = [1.0] + [0.0] * d
    facs = [[None] * d] + [[D if k == t else None for k in range(d)] for t in range(d)]
    tabs = oim.build_tables(facs, eta, zeta, [q] * d)
    ref, _, _ = oim.step(f0, tabs, sweeps, w["lam"])
    pert, _, _ = oim.step(perturb(f0), tabs, sweeps, w["lam"])
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=1.0, schedule="gauss-seidel",
                                 lam=w["lam"])
    out = implicit.step(cp.CPTensor(S, f0), pair, None, cfg).to_numpy()
    return metrics.cp_rel_diff(ref, out), metrics.cp_rel_diff(ref, pert), "one step, 3 GS sweeps (state perturbed)"


def cfg4():
    w = workloads.cfg4(0, batch=1)
    d, Q, k = w["d"], w["Q"], w["k"]
    nodes = oht.balanced_tree(d)
    frames, transfers, li, ii = [None] * len(nodes), [None] * len(nodes), 0, 0
    for t, nd in enumerate(nodes):
        if oht.is_leaf(nd):
            frames[t] = w["frames"][0, li]
            li += 1
        else:
            transfers[t] = w["transfers"][0, ii][:, :, :1] if t == 0 else w["transfers"][0, ii]
            ii += 1
    h = (nodes, frames, transfers)
    ref, _ = oht.truncate(h, 16, 0.0)
    hp = (nodes, [None if f is None else perturb([f])[0] for f in frames], transfers)
    pert, _ = oht.truncate(hp, 16, 0.0)
    specs = tuple(BasisSpec(Q, 1.0, "collocation") for _ in range(d))
    out, _ = ht.truncate(ht.HTTensor(specs, ht.balanced_tree(d), frames, transfers), 16, 0.0)
    return metrics.ht_rel_diff(ref, out.to_oracle()), metrics.ht_rel_diff(ref, pert), "one tensor (leaf frames perturbed)"


RUNS = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}

if __name__ == "__main__":
    print(f"{'config':6s} {'gpu vs oracle':>14s} {'oracle vs 1e-13-perturbed oracle':>34s}   run")
    for name in sys.argv[1:] or list(RUNS):
        t0 = time.time()
        g, p, what = RUNS[name]()
        print(f"{name:6s} {g:14.2e} {p:34.2e}   {what} ({time.time() - t0:.0f} s)", flush=True)
