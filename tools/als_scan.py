"""Scan fused-ALS time per mode update over problem sizes (device-resident, CUDA events)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, workloads  # noqa: E402


def t_mode(d, Q, R, r, grid, sweeps=10):
    w = workloads.cfg1(0, d=d, Q=Q, R=R, r=r)
    T = cp.CPTensor(w["specs"], w["V"])
    I0 = cp.CPTensor(w["specs"], w["init"])
    info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10, grid=grid)
    U = I0.data.clone()
    for _ in range(2):
        cp._als_device(T, U, r, cfg, None, info)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        cp._als_device(T, U, r, cfg, None, info)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    return ms * 1e3 / (sweeps * d)


if __name__ == "__main__":
    cases = [(6, 256, 512, 32, 128), (6, 256, 512, 8, 128), (6, 256, 512, 32, 8), (6, 32, 64, 8, 8),
             (6, 32, 64, 8, 1), (2, 16, 16, 2, 1), (6, 64, 128, 16, 32), (6, 256, 512, 16, 128)]
    for c in cases:
        print(f"d={c[0]} Q={c[1]} R={c[2]} r={c[3]} grid={c[4]}: {t_mode(*c):8.2f} us per mode update", flush=True)
