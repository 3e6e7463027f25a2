"""A few config-0 explicit steps (for launch lists): python tools/cfg0_once.py [steps] [cfg0|cfg3]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, explicit, operators, workloads  # noqa: E402
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
which = sys.argv[2] if len(sys.argv) > 2 else "cfg0"
if which == "cfg0":
    w = workloads.cfg0(0)
    L = operators.advection_operator(w["a"], w["specs"])
    f0 = cp.CPTensor(w["specs"], w["ic"]["factors"])
else:
    w = workloads.cfg3(0)
    L = operators.SeparableOperator(w["specs"], tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
    f0 = cp.CPTensor(w["specs"], w["factors"])
cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused",
                              als=cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"]))
out = explicit.run(f0, L, cfg, steps)
torch.cuda.synchronize()
print("ok", float(out.data.norm()))
