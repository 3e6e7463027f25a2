"""A/B timing of ALS kernel variants via debug hooks (ns cap, skip mask)."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_skip.argtypes = [ctypes.c_int]
L.tp_debug_set_als_ns.argtypes = [ctypes.c_int]
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 256
R = int(sys.argv[2]) if len(sys.argv) > 2 else 512
r = int(sys.argv[3]) if len(sys.argv) > 3 else 32
w = workloads.cfg1(0, Q=Q, R=R, r=r)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)


def t(ns, skip, grid=0, sweeps=20):
    L.tp_debug_set_als_ns(ns)
    L.tp_debug_set_als_skip(skip)
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10, grid=grid)
    U = I0.data.clone()
    for _ in range(2):
        U.copy_(I0.data); cp._als_device(T, U, r, cfg, None, info)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        U.copy_(I0.data); cp._als_device(T, U, r, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    L.tp_debug_set_als_ns(6); L.tp_debug_set_als_skip(0)
    return e0.elapsed_time(e1) / 5 * 1e3 / (sweeps * 6)


print(f"Q={Q} R={R} r={r}")
for nm, ns, sk in [("NS on", 6, 0), ("NS off (sweep)", 0, 0), ("skip inverse", 6, 1), ("skip all but syncs", 6, 127)]:
    print(f"{nm:20s} {t(ns, sk):7.2f} us/mode", flush=True)
for sw in (1, 2, 5):
    print(f"sweeps={sw:2d} NS on {t(6, 0, sweeps=sw):7.2f}  off {t(0, 0, sweeps=sw):7.2f} us/mode", flush=True)

ALL = 127
print("add-back from the skeleton (all phases skipped):")
base = t(6, ALL)
for nm, bit in [("inverse NS", 1), ("stage_u", 2), ("cross", 4), ("gram_share", 8), ("Y gemm/store", 16),
                ("slice fetch", 32), ("reduce", 64)]:
    print(f"  + {nm:16s} {t(6, ALL & ~bit) - base:+7.2f} us/mode")
print(f"  + inverse sweep    {t(0, ALL & ~1) - base:+7.2f} us/mode")
