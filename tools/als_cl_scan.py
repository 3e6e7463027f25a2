"""ALS variant/grid scan on random targets: python tools/als_cl_scan.py Q R r sweeps [var:grid ...]
var: 0 auto, 1 persistent, 2 cluster (grid = cluster size), 3 small, 4 persistent-as-one-cluster."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402
from oracle import metrics  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
Q, R, r, sweeps = (int(x) for x in sys.argv[1:5])
combos = [tuple(int(v) for v in c.split(":")) for c in sys.argv[5:]] or [(0, 0)]
d = 6
rng = np.random.default_rng(0)
specs = tuple(BasisSpec(Q, np.pi, "collocation", lo=0.0) for _ in range(d))
V = [rng.standard_normal((Q, R)) / np.sqrt(Q) for _ in range(d)]
T = cp.CPTensor(specs, V)
I0 = cp.CPTensor(specs, [v[:, :r].copy() for v in V])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
U = I0.data.clone()
ref = None
for var, g in combos:
    if var == 2:
        L.tp_debug_set_als_variant(2, g); grid = 0
    else:
        L.tp_debug_set_als_variant(var, 0); grid = g
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10, grid=grid)
    try:
        plan = cp.als_plan([Q] * d, R, r, grid)
        for _ in range(2):
            U.copy_(I0.data); cp._als_device(T, U, r, cfg, None, info)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(var, g, "failed:", e, flush=True)
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        U.copy_(I0.data); cp._als_device(T, U, r, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    out = cp.CPTensor(specs, data=U.clone(), rank=r).to_numpy()
    if ref is None:
        ref = out
    rel = metrics.cp_rel_diff(ref, out)
    print(f"var {var} grid {g:3d} plan {plan}: {ms*1e3:8.1f} us/trunc {ms*1e3/(6*sweeps):6.2f} us/mode "
          f"info={info.tolist()} rel {rel:.2e}", flush=True)
L.tp_debug_set_als_variant(0, 0)
