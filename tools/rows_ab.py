"""A/B of cluster-row kernel schedules on the same box (alternating, config 1)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402
L = _lib.lib()
for f in ("tp_debug_set_als_rows_mc", "tp_debug_set_als_rows_split"):
    getattr(L, f).argtypes = [ctypes.c_int]
w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
U = I0.data.clone()
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
modes = {"split": (1, 1), "unsplit": (1, 0)}
res = {k: [] for k in modes}
for rep in range(6):
    for name, (mc, gp) in modes.items():
        L.tp_debug_set_als_rows_mc(mc)
        L.tp_debug_set_als_rows_split(gp)
        for _ in range(2):
            U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            U.copy_(I0.data)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); cp._als_device(T, U, 32, cfg, None, info); e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name].append(float(np.median(ts)))
L.tp_debug_set_als_rows_mc(1)
L.tp_debug_set_als_rows_split(1)
for k, v in res.items():
    print(f"{k:9s} median {np.median(v) * 1e3:7.1f} us  runs {['%.0f' % (x * 1e3) for x in v]}")
