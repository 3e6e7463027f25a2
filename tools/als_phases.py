"""Per-phase clock64 breakdown of the fused ALS kernel (CTA 0) via the debug hook."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402

NAMES = ["A:gram (after cross)", "A:had+Y", "sync1", "B:loadG", "B:chol||reduce", "B:solve+write", "sync2",
         "(unused)", "warp0 invert", "warp1 reduce", "A:stage_u", "A:cross"]


def run(grid, Q=256, R=512, r=32):
    w = workloads.cfg1(0, Q=Q, R=R, r=r)
    T = cp.CPTensor(w["specs"], w["V"])
    I0 = cp.CPTensor(w["specs"], w["init"])
    dev = T.data.device
    prof = torch.zeros(16, dtype=torch.int64, device=dev)
    L = _lib.lib()
    L.tp_debug_set_als_profile.argtypes = [ctypes.c_void_p]
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10, grid=grid)
    U = I0.data.clone()
    cp._als_device(T, U, r, cfg, None, info)
    L.tp_debug_set_als_profile(prof.data_ptr())
    U.copy_(I0.data)
    cp._als_device(T, U, r, cfg, None, info)
    torch.cuda.synchronize()
    L.tp_debug_set_als_profile(None)
    p = prof.cpu().numpy() / 120.0
    tot = p[[0, 1, 2, 3, 4, 5, 6, 10, 11]].sum()
    print(f"grid={grid} Q={Q} R={R} r={r}: cycles per mode update (CTA 0): total {tot:.0f}")
    for i in [10, 11, 0, 1, 2, 3, 4, 5, 6]:
        print(f"   {NAMES[i]:22s} {p[i]:9.0f}  ({100*p[i]/tot:4.1f}%)")
    raw = prof.cpu().numpy()
    print(f"   Newton-Schulz accepted {raw[14]}, fell back {raw[15]}")


if __name__ == "__main__":
    run(0)
