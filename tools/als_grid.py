"""Config-1 ALS truncation time vs persistent grid size."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, workloads  # noqa: E402

w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
U = I0.data.clone()
for g in [int(x) for x in sys.argv[1:]] or [0, 16, 32, 48, 64, 84, 100, 128, 148]:
    cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10, grid=g)
    for _ in range(2):
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"grid {g:4d}: {ms*1e3:8.1f} us/truncation {20/ms*1e3:8.0f} sweeps/s {ms*1e3/120:6.2f} us/mode", flush=True)
