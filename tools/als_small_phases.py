"""Phase clock64 totals of als_small (config 0 size): python tools/als_small_phases.py [Q R r sweeps]"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp
from paper_1803_10270_b200.basis import BasisSpec
Q, R, r, sw = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 78, 6, 10)))
rng = np.random.default_rng(0)
V = [rng.standard_normal((Q, R)) / np.sqrt(Q) for _ in range(6)]
S = tuple(BasisSpec(Q, np.pi, "collocation", lo=0.0) for _ in range(6))
T, I0 = cp.CPTensor(S, V), cp.CPTensor(S, [v[:, :r].copy() for v in V])
L = _lib.lib(); L.tp_debug_set_als_profile.argtypes = [ctypes.c_void_p]
prof = torch.zeros(32, dtype=torch.int64, device="cuda")
cfg = cp.ALSApproxConfig(max_sweeps=sw, stall=-np.inf, reg=1e-10)
cp.cp_approx_als(T, r, cfg, init=I0)
L.tp_debug_set_als_profile(prof.data_ptr())
cp.cp_approx_als(T, r, cfg, init=I0)
torch.cuda.synchronize()
L.tp_debug_set_als_profile(None)
p = prof.cpu().numpy()[:6] / (6.0 * sw)
names = ["-", "-", "U_j", "refresh+next(had,rhs | G,inverse)", "(warp-0 path)", "loop head"]
print(f"cycles per mode update: total {p.sum() - p[4]:.0f}")
for n, v in zip(names, p):
    print(f"  {n:12s} {v:7.0f}")
