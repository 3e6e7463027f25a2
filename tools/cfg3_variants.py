"""Config-3 fused-AB2 trajectory time per ALS kernel choice (default plan vs cluster-row kernel)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, explicit, operators, workloads  # noqa: E402
L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
L.tp_debug_set_als_rows.argtypes = [ctypes.c_int, ctypes.c_int]
w = workloads.cfg3(0)
S = w["specs"]
op = operators.SeparableOperator(S, tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                              als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
f0 = cp.CPTensor(S, w["factors"])
steps = 40
ref = None
for name, var, cs, pr in [("default", 0, 0, 0), ("rows16 P1", 8, 16, 1), ("rows16 P2", 8, 16, 2), ("rows8 P2", 8, 8, 2),
                          ("rows8 P4", 8, 8, 4), ("rows16 P4", 8, 16, 4)]:
    L.tp_debug_set_als_variant(var, cs)
    L.tp_debug_set_als_rows(1, pr)
    try:
        out = explicit.run(f0, op, cfg, 4)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = explicit.run(f0, op, cfg, steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ref is None:
            ref = out
        from oracle import metrics
        rel = metrics.cp_rel_diff(ref.to_numpy(), out.to_numpy())
        print(f"{name:10s} {steps / ms * 1e3:8.1f} steps/s  rel vs default {rel:.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "failed", e, flush=True)
L.tp_debug_set_als_variant(0, 0)
L.tp_debug_set_als_rows(1, 0)
