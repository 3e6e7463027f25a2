import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp
from paper_1803_10270_b200.basis import BasisSpec
from oracle import metrics, cp_als as ocp
L = _lib.lib(); L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
g = np.load("tests/golden/cp_als.npz"); n = "r32_q64"
V = [g[f"{n}_V_{k}"] for k in range(4)]; I = [g[f"{n}_init_{k}"] for k in range(4)]
S = tuple(BasisSpec(64, np.pi, "collocation", lo=0.0) for _ in range(4))
ref = ocp.als(V, I, 6, lam=1e-10)
var, grid, ns = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
L.tp_debug_set_als_variant(var, 0)
L.tp_debug_set_als_ns(ns)
for tr in ([], [], None):
    out = cp.cp_approx_als(cp.CPTensor(S, V), 32, cp.ALSApproxConfig(max_sweeps=6, stall=-np.inf, reg=1e-10, grid=grid), init=cp.CPTensor(S, I), trace=tr)
    print(var, grid, ns, tr is not None, "vs oracle %.2e" % metrics.cp_rel_diff(ref, out.to_numpy()), (tr or [0])[0], flush=True)
