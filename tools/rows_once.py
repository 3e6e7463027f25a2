"""One config-1 truncation on the cluster-row kernel (variant 8), for ncu."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
L.tp_debug_set_als_rows.argtypes = [ctypes.c_int, ctypes.c_int]
L.tp_debug_set_als_variant(8, int(sys.argv[1]) if len(sys.argv) > 1 else 16)
L.tp_debug_set_als_rows(1, 0)
w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
U = I0.data.clone()
cp._als_device(T, U, 32, cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10), None, info)
torch.cuda.synchronize()
print("info", info.tolist())
