"""Per-phase clock64 breakdown of the fused ALS kernel (CTA 0) via the debug hook."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402

NAMES = ["(loop head)", "A:gram_share", "A:had+Y", "barrier1", "B:reduce", "B:wait Y slices", "B:write U",
         "barrier2", "B:wait G/X", "B:solve (NS/exact)", "A:stage_u", "A:cross", "A:exchange", "-", "-", "-"]


def run(grid, Q=256, R=512, r=32, sweeps=20):
    w = workloads.cfg1(0, Q=Q, R=R, r=r)
    T = cp.CPTensor(w["specs"], w["V"])
    I0 = cp.CPTensor(w["specs"], w["init"])
    dev = T.data.device
    prof = torch.zeros(32, dtype=torch.int64, device=dev)
    L = _lib.lib()
    L.tp_debug_set_als_profile.argtypes = [ctypes.c_void_p]
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10, grid=grid)
    U = I0.data.clone()
    cp._als_device(T, U, r, cfg, None, info)
    L.tp_debug_set_als_profile(prof.data_ptr())
    U.copy_(I0.data)
    cp._als_device(T, U, r, cfg, None, info)
    torch.cuda.synchronize()
    L.tp_debug_set_als_profile(None)
    p = prof.cpu().numpy() / (sweeps * 6.0)
    tot = p[:16].sum()
    print(f"grid={grid} Q={Q} R={R} r={r}: cycles per mode update (CTA 0): total {tot:.0f}")
    for i in [0, 10, 11, 12, 1, 2, 3, 8, 5, 4, 9, 6, 7]:
        print(f"   {NAMES[i]:22s} {p[i]:9.0f}  ({100*p[i]/tot:4.1f}%)")
    raw = prof.cpu().numpy()


if __name__ == "__main__":
    import os
    Lb = _lib.lib()
    Lb.tp_debug_set_als_ns.argtypes = [ctypes.c_int]
    Lb.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
    var = [int(x) for x in os.environ.get("ALS_VARIANT", "0,0").split(",")]
    Lb.tp_debug_set_als_variant(var[0], var[1])
    Lb.tp_debug_set_als_profile_cta.argtypes = [ctypes.c_int]
    Lb.tp_debug_set_als_profile_cta(int(os.environ.get("ALS_PROF_CTA", "0")))
    for ns in (6,):
        print(f"--- Newton-Schulz cap {ns}")
        Lb.tp_debug_set_als_ns(ns)
        size = [int(x) for x in os.environ.get("ALS_SIZE", "256,512,32,20").split(",")]
        for g in [int(x) for x in sys.argv[1:]] or [0]:
            run(g, *size)
