"""Time the fused ALS kernel with phases skipped (debug mask) -> phase cost by subtraction."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_skip.argtypes = [ctypes.c_int]
w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
U = I0.data.clone()
names = {0: "full", 1: "-inverse", 2: "-stage_u", 4: "-cross", 8: "-gram_share", 16: "-Y gemm/store",
         32: "-phaseB slice fetch", 64: "-reduce", 1 | 2 | 4 | 8 | 16 | 32 | 64: "-all (syncs+rest)"}
base = None
for mask, nm in names.items():
    L.tp_debug_set_als_skip(mask)
    for _ in range(2):
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 5 * 1e3 / 120
    base = us if base is None else base
    print(f"{nm:22s} {us:7.2f} us/mode update   (delta {base - us:+6.2f})", flush=True)
L.tp_debug_set_als_skip(0)
