"""Device-resident timing of every BASELINE config through the public API."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, explicit, implicit, operators, workloads  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def time_it(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def cfg0(steps):
    w = workloads.cfg0(0)
    S = w["specs"]
    L = operators.advection_operator(w["a"], S)
    cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                  als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
    f0 = cp.CPTensor(S, w["ic"]["factors"])
    ms, _ = time_it(lambda: explicit.run(f0, L, cfg, steps))
    print(f"cfg0: {steps} steps in {ms:.1f} ms -> {steps / ms * 1e3:.0f} steps/s", flush=True)


def cfg3(steps):
    w = workloads.cfg3(0)
    S = w["specs"]
    L = operators.SeparableOperator(S, tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
    cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                                  als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
    f0 = cp.CPTensor(S, w["factors"])
    ms, _ = time_it(lambda: explicit.run(f0, L, cfg, steps))
    print(f"cfg3: {steps} steps in {ms:.1f} ms -> {steps / ms * 1e3:.0f} steps/s", flush=True)


def cfg2(steps):
    w = workloads.cfg2(0)
    S = w["specs"]
    L = operators.advection_operator(w["a"], S)
    pair = operators.implicit_euler_pair(L, w["dt"])
    cfg = implicit.ALSStepConfig(dt=w["dt"], eps_tol=0.0, max_sweeps=w["sweeps"], delta_beta=1.0,
                                 schedule="gauss-seidel", lam=w["lam"])
    f0 = cp.CPTensor(S, w["ic"]["factors"])
    ws = implicit.StepWorkspace(pair, cfg)
    ms, _ = time_it(lambda: implicit.run(f0, pair, cfg, steps, workspace=ws))
    print(f"cfg2: {steps} steps in {ms:.1f} ms -> {steps / ms * 1e3:.2f} steps/s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg0", "cfg3", "cfg2"]
    if "cfg0" in which:
        cfg0(100)
    if "cfg3" in which:
        cfg3(50)
    if "cfg2" in which:
        cfg2(3)
