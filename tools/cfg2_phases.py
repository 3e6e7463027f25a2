"""cfg2 fused circulant step: per-phase clock64 split of CTA 0 (debug hook)."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, implicit, operators, workloads  # noqa: E402
L = _lib.lib()
L.tp_debug_set_circ_prof.argtypes = [ctypes.c_void_p]
w = workloads.cfg2(0)
pair = operators.implicit_euler_pair(operators.advection_operator(w["a"], w["specs"]), w["dt"])
cfg = implicit.ALSStepConfig(dt=w["dt"], eps_tol=0.0, max_sweeps=w["sweeps"], delta_beta=1.0,
                             schedule="gauss-seidel", lam=w["lam"])
f0 = cp.CPTensor(w["specs"], w["ic"]["factors"])
implicit.step(f0, pair, None, cfg)
prof = torch.zeros(16, dtype=torch.int64, device="cuda")
L.tp_debug_set_circ_prof(prof.data_ptr())
implicit.step(f0, pair, None, cfg)
torch.cuda.synchronize()
L.tp_debug_set_circ_prof(None)
n = 6 * w["sweeps"]
names = ["loop/start", "F load", "F gamma+M", "F chol+solve", "F conv", "F gram terms", "barrier 1",
         "E H (after reduce)", "barrier 2", "E reduce"]
p = prof.cpu().tolist()
tot = sum(p[:10])
for i, nm in enumerate(names):
    print(f"{nm:16s} {p[i] / n:9.0f} cycles/mode-update")
print(f"{'total':16s} {tot / n:9.0f}")
