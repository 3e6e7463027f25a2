"""One config-2 implicit step on the DENSE solver (normal-equation assembly + blocked Cholesky), for ncu."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, implicit, operators, workloads  # noqa: E402
w = workloads.cfg2(0)
pair = operators.implicit_euler_pair(operators.advection_operator(w["a"], w["specs"]), w["dt"])
cfg = implicit.ALSStepConfig(dt=w["dt"], eps_tol=0.0, max_sweeps=int(sys.argv[1]) if len(sys.argv) > 1 else 1,
                             delta_beta=1.0, schedule="gauss-seidel", lam=w["lam"], solver="dense")
f0 = cp.CPTensor(w["specs"], w["ic"]["factors"])
f = implicit.step(f0, pair, None, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f = implicit.step(f0, pair, None, cfg)
e1.record()
torch.cuda.synchronize()
print("ok", float(f.data.norm()), "ms per step (%d sweeps):" % cfg.max_sweeps, e0.elapsed_time(e1))
if len(sys.argv) > 2:
    import ctypes
    from paper_1803_10270_b200 import _lib
    Lb = _lib.lib()
    Lb.tp_debug_set_dense_prof.argtypes = [ctypes.c_void_p]
    prof = torch.zeros(8, dtype=torch.int64, device="cuda")
    Lb.tp_debug_set_dense_prof(prof.data_ptr())
    implicit.step(f0, pair, None, cfg)
    torch.cuda.synchronize()
    Lb.tp_debug_set_dense_prof(None)
    p = prof.cpu().numpy()
    print("diag kernel cycles: load %.0f | factor %.0f | inverse+store %.0f (per call, %d calls)" %
          (p[0] / p[3], p[1] / p[3], p[2] / p[3], p[3]))
