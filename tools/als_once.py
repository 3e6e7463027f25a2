"""One config-1 truncation (for ncu): python tools/als_once.py [grid]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, workloads  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 0
w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
out = cp.cp_approx_als(T, 32, cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10, grid=g), init=I0)
torch.cuda.synchronize()
print("ok", float(out.data.norm()))
