"""Time one config-3 truncation on a real AB2 target (vs the random-target scan)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import cp, explicit, operators, workloads  # noqa: E402
w = workloads.cfg3(0)
S = w["specs"]
L = operators.SeparableOperator(S, tuple(w["weights"]), tuple(tuple(m) for m in w["mats"]))
als = cp.ALSApproxConfig(max_sweeps=w["sweeps"], stall=-np.inf, reg=w["lam"])
cfg = explicit.ExplicitConfig(dt=w["dt"], r_max=w["r"], recipe="fused", als=als)
f0 = cp.CPTensor(S, w["factors"])
f1 = explicit.run(f0, L, cfg, 3, graph=False)
f2 = explicit.run(f0, L, cfg, 4, graph=False)
tgt = explicit.ab2_target(f1, f2, L, w["dt"])
print("target rank", tgt.rank, cp.als_plan(tgt.qs, tgt.rank, w["r"]))
info = torch.zeros(2, dtype=torch.int32, device="cuda")
U = f2.data.clone()
for name, T in [("real", tgt)]:
    for _ in range(3):
        U.copy_(f2.data); cp._als_device(T, U, w["r"], als, None, info)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        U.copy_(f2.data); cp._als_device(T, U, w["r"], als, None, info)
    e1.record(); torch.cuda.synchronize()
    print(name, f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us per truncation", info.tolist())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    t2 = explicit.ab2_target(f1, f2, L, w["dt"])
e1.record(); torch.cuda.synchronize()
print(f"ab2_target {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
torch.cuda.synchronize()
import time
t0 = time.perf_counter(); out = explicit.run(f0, L, cfg, 50); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"run 50 steps {1e3*(t1-t0):.1f} ms -> {(t1-t0)/50*1e6:.0f} us/step")
import ctypes
from paper_1803_10270_b200 import _lib  # noqa: E402
Lb = _lib.lib()
Lb.tp_debug_set_als_profile.argtypes = [ctypes.c_void_p]
Lb.tp_debug_set_als_ns.argtypes = [ctypes.c_int]
NAMES = ["(loop head)", "A:gram_share", "A:had+Y", "barrier1", "B:reduce", "B:wait Y slices", "B:write U",
         "barrier2", "B:wait G/X", "B:solve (NS/exact)", "A:stage_u", "A:cross", "A:exchange", "-", "-", "-"]
for label, T, U0 in [("real", tgt, f2.data), ("random", None, None)]:
    if T is None:
        rng = np.random.default_rng(0)
        V = [rng.standard_normal((64, 588)) / 8 for _ in range(6)]
        T = cp.CPTensor(S, V)
        U0 = cp.CPTensor(S, [v[:, :12].copy() for v in V]).data
    for ns in (6, 0):
        Lb.tp_debug_set_als_ns(ns)
        prof = torch.zeros(32, dtype=torch.int64, device="cuda")
        U.copy_(U0); cp._als_device(T, U, w["r"], als, None, info)
        Lb.tp_debug_set_als_profile(prof.data_ptr())
        U.copy_(U0); cp._als_device(T, U, w["r"], als, None, info)
        torch.cuda.synchronize()
        Lb.tp_debug_set_als_profile(None)
        p = prof.cpu().numpy() / 60.0
        print(label, "ns", ns, f"total {p[:16].sum():.0f}", " ".join(f"{NAMES[i]}={p[i]:.0f}" for i in [10, 11, 1, 2, 3, 8, 4, 9, 6, 7]))
Lb.tp_debug_set_als_ns(6)
Lb.tp_debug_set_als_early_inv.argtypes = [ctypes.c_int]
for ei in (1, 0, 1):
    Lb.tp_debug_set_als_early_inv(ei)
    for _ in range(3):
        U.copy_(f2.data); cp._als_device(tgt, U, w["r"], als, None, info)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        U.copy_(f2.data); cp._als_device(tgt, U, w["r"], als, None, info)
    e1.record(); torch.cuda.synchronize()
    print("early_inv", ei, f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us per truncation", info.tolist(), cp.als_plan(tgt.qs, tgt.rank, w["r"]))
