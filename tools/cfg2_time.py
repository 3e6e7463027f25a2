"""cfg2: time a run of implicit steps (device-resident), fused vs per-kernel circulant path."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, implicit, operators, workloads  # noqa: E402
L = _lib.lib()
L.tp_debug_set_circ_fused.argtypes = [ctypes.c_int]
w = workloads.cfg2(0)
pair = operators.implicit_euler_pair(operators.advection_operator(w["a"], w["specs"]), w["dt"])
cfg = implicit.ALSStepConfig(dt=w["dt"], eps_tol=0.0, max_sweeps=w["sweeps"], delta_beta=1.0,
                             schedule="gauss-seidel", lam=w["lam"])
ws = implicit.StepWorkspace(pair, cfg)
f0 = cp.CPTensor(w["specs"], w["ic"]["factors"])
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for fused in [1, 0, 1]:
    L.tp_debug_set_circ_fused(fused)
    implicit.run(f0, pair, cfg, 2, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = implicit.run(f0, pair, cfg, n, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"fused={fused}: {ms:.3f} ms/step -> {1e3 / ms:.1f} steps/s  |f|={float(out.data.norm()):.12f}", flush=True)
