import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, implicit, operators, workloads  # noqa: E402
w = workloads.cfg2(0)
pair = operators.implicit_euler_pair(operators.advection_operator(w["a"], w["specs"]), w["dt"])
cfg = implicit.ALSStepConfig(dt=w["dt"], eps_tol=0.0, max_sweeps=int(sys.argv[1]) if len(sys.argv) > 1 else 2,
                             delta_beta=1.0, schedule="gauss-seidel", lam=w["lam"])
f = implicit.step(cp.CPTensor(w["specs"], w["ic"]["factors"]), pair, None, cfg)
torch.cuda.synchronize()
print("ok", float(f.data.norm()))
