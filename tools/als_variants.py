"""Config-1 ALS: persistent vs cluster variants (timing + agreement)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402
from oracle import metrics  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
U = I0.data.clone()
outs = {}
for name, var, cs in [("persistent", 1, 0), ("cluster8", 2, 8), ("cluster4", 2, 4), ("cluster2", 2, 2)]:
    L.tp_debug_set_als_variant(var, cs)
    try:
        for _ in range(2):
            U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(name, "failed:", e)
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    outs[name] = cp.CPTensor(w["specs"], data=U.clone(), rank=32).to_numpy()
    rel = metrics.cp_rel_diff(outs["persistent"], outs[name]) if "persistent" in outs else float("nan")
    print(f"{name:11s} {ms*1e3:8.1f} us/truncation {20/ms*1e3:8.0f} sweeps/s  info={info.tolist()}  rel vs persistent {rel:.2e}", flush=True)
L.tp_debug_set_als_variant(0, 0)
