"""ALS time per truncation for a given size across kernel variants / grids:
python tools/als_size_variants.py Q R r sweeps"""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402

Q, R, r, sweeps = (int(x) for x in sys.argv[1:5])
L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
w = workloads.cfg1(0, Q=Q, R=R, r=r)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
U = I0.data.clone()
for name, var, cs, grid in [("auto", 0, 0, 0), ("small", 3, 0, 0), ("persistent g=1", 1, 0, 1), ("persistent g=4", 1, 0, 4),
                            ("persistent g=12", 1, 0, 12), ("persistent g=32", 1, 0, 32), ("persistent g=64", 1, 0, 64),
                            ("cluster2", 2, 2, 0), ("cluster4", 2, 4, 0), ("cluster8", 2, 8, 0)]:
    L.tp_debug_set_als_variant(var, cs)
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10, grid=grid)
    try:
        plan = cp.als_plan([Q] * 6, R, r, grid)
        for _ in range(2):
            U.copy_(I0.data); cp._als_device(T, U, r, cfg, None, info)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(f"{name:16s} failed: {e}")
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        U.copy_(I0.data); cp._als_device(T, U, r, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:16s} {ms*1e3:8.1f} us/truncation  {ms*1e3/(6*sweeps):6.2f} us/mode  plan {plan}", flush=True)
L.tp_debug_set_als_variant(0, 0)
