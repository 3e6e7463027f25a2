"""Quick device timing of the fused ALS kernel at BASELINE config 1 over grid sizes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402


def main():
    w = workloads.cfg1(0)
    S = w["specs"]
    T = cp.CPTensor(S, w["V"])
    I0 = cp.CPTensor(S, w["init"])
    dev = T.data.device
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    grids = [int(x) for x in sys.argv[1:]] or [0, 16, 32, 64, 96, 128, 148]
    for trace_on in (False, True):
        for g in grids:
            cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10, grid=g)
            tb = torch.zeros(20, dtype=torch.float64, device=dev) if trace_on else None
            U = I0.data.clone()
            for _ in range(3):
                U.copy_(I0.data)
                cp._als_device(T, U, 32, cfg, tb, info)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 10
            e0.record()
            for _ in range(n):
                cp._als_device(T, U, 32, cfg, tb, info)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            print(f"trace={trace_on} grid={g:4d}  {ms*1e3:9.1f} us/truncation  {20/ms*1e3:10.0f} sweeps/s  info={info.tolist()}")
    t0 = time.perf_counter()
    from oracle import cp_als as ocp
    ocp.als(w["V"], w["init"], 20, lam=1e-10)
    print(f"oracle numpy real fp64: {(time.perf_counter()-t0)*1e3:.1f} ms")


if __name__ == "__main__":
    main()
