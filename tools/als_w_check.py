"""Gram-space ALS kernel (variant 9) against the oracle and the cluster-row kernel (variant 8):
parity on config 1 and on ragged / small shapes, conditioning fallback, timings.
python tools/als_w_check.py [quick]"""
import ctypes
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import cp_als as ocp, metrics  # noqa: E402
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
L.tp_debug_set_als_w.argtypes = [ctypes.c_int, ctypes.c_double]


def specs(qs):
    return tuple(BasisSpec(q, 1.0, "collocation") for q in qs)


def run(V, init, sweeps, reg, variant, trace=None):
    L.tp_debug_set_als_variant(variant, 0)
    qs = [v.shape[0] for v in V]
    S = specs(qs)
    plan = cp.als_plan(qs, V[0].shape[1], init[0].shape[1])
    out = cp.cp_approx_als(cp.CPTensor(S, V), init[0].shape[1],
                           cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=reg), init=cp.CPTensor(S, init),
                           trace=trace)
    torch.cuda.synchronize()
    return out, plan["kernel"]


def timeit(V, init, sweeps, reg, variant, n=20):
    L.tp_debug_set_als_variant(variant, 0)
    qs = [v.shape[0] for v in V]
    S = specs(qs)
    T, I0 = cp.CPTensor(S, V), cp.CPTensor(S, init)
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=reg)
    for _ in range(3):
        cp.cp_approx_als(T, init[0].shape[1], cfg, init=I0, sync=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        cp.cp_approx_als(T, init[0].shape[1], cfg, init=I0, sync=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


w = workloads.cfg1(0)
V, init = w["V"], w["init"]
ref = ocp.als(V, init, 20, lam=1e-10)
for variant in (8, 9):
    out, k = run(V, init, 20, 1e-10, variant)
    print(f"cfg1 variant {variant} ({k}): rel vs oracle {metrics.cp_rel_diff(ref, out.to_numpy()):.3e}", flush=True)
tr, otr = [], []
out, k = run(V, init, 6, 1e-10, 9, trace=tr)
ref6 = ocp.als(V, init, 6, lam=1e-10, trace=otr)
print(f"cfg1 traced 6 sweeps ({k}): rel {metrics.cp_rel_diff(ref6, out.to_numpy()):.3e} trace err "
      f"{np.max(np.abs(np.array(tr) - np.array(otr))):.3e} of {otr[-1]:.3e}", flush=True)
for variant in (8, 9):
    print(f"cfg1 variant {variant}: {timeit(V, init, 20, 1e-10, variant):.1f} us per truncation", flush=True)
L.tp_debug_set_als_w_pair.argtypes = [ctypes.c_int]
L.tp_debug_set_als_w_pair(0)
out, k = run(V, init, 20, 1e-10, 9)
print(f"cfg1 variant 9 without CTA pairs ({cp.als_plan([v.shape[0] for v in V], 512, 32)}): rel vs oracle "
      f"{metrics.cp_rel_diff(ref, out.to_numpy()):.3e}, {timeit(V, init, 20, 1e-10, 9):.1f} us per truncation", flush=True)
L.tp_debug_set_als_w_pair(1)
print(f"plan with pairs: {cp.als_plan([v.shape[0] for v in V], 512, 32)}", flush=True)
L.tp_debug_set_als_profile.argtypes = [ctypes.c_void_p]
names = ["top", "reduce M (wait + sum)", "reduced M wait + load", "G step", "A + Newton-Schulz residual", "join wait",
         "exact inverse", "C / X1 / M / publish", "gemm (wait+load+mma)", "T reduce", "join wait (gemm)", "(gemm) rest of round",
         "setup (x120: one-off)", "tail (x120)", "final phase (x120: one-off)"]
if True:
    prof = torch.zeros(48, dtype=torch.int64, device="cuda")
    L.tp_debug_set_als_profile(prof.data_ptr())
    run(V, init, 20, 1e-10, 9)
    L.tp_debug_set_als_profile(None)
    p = prof.cpu().numpy() / 120.0
    print(f"cycles per mode update (CTA 0; A group thread 128 | GEMM group thread 0), {timeit(V, init, 20, 1e-10, 9):.1f} us per truncation:")
    for n_, v in zip(names, p):
        print(f"  {n_:28s} {v:9.0f}")
    ab = prof.cpu().numpy()[16:48]
    t0 = ab[ab > 0].min()
    ev = sorted((int(v - t0), f"r{61 + i // 16} {names[i % 16] if i % 16 < len(names) else i % 16}") for i, v in enumerate(ab) if v > 0)
    print("  timeline (rounds 61-62): " + " | ".join(f"{t}: {n}" for t, n in ev))
if len(sys.argv) > 1:
    sys.exit(0)
rng = np.random.default_rng(3)
for qs, R, r, reg in [((256,) * 6, 512, 32, None), ((100, 90, 120, 80), 300, 20, 1e-10), ((80, 70, 96), 257, 7, None),
                      ((300, 280), 1000, 32, 1e-10), ((128,) * 8, 400, 13, 1e-10)]:
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    tr, otr = [], []
    out, k = run(V, init, 5, reg, 0, trace=tr)
    ref = ocp.als(V, init, 5, lam=reg, trace=otr)
    print(f"{qs} R={R} r={r} reg={reg} ({k}): rel {metrics.cp_rel_diff(ref, out.to_numpy()):.3e} trace err "
          f"{np.max(np.abs(np.array(tr) - np.array(otr))):.3e}", flush=True)
# ill-conditioned: two equal init columns -> the fallback must rerun the truncation
qs, R, r = (96, 80, 100, 90), 320, 8
V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
init = [v[:, :r].copy() for v in V]
for f in init:
    f[:, 1] = f[:, 0] * (1.0 + 1e-9)
out, k = run(V, init, 4, 1e-10, 0)
ref = ocp.als(V, init, 4, lam=1e-10)
out8, _ = run(V, init, 4, 1e-10, 8)
print(f"ill-conditioned ({k}): rel vs oracle {metrics.cp_rel_diff(ref, out.to_numpy()):.3e}, bitwise equal to "
      f"als_rows: {torch.equal(out.data, out8.data)}", flush=True)
L.tp_debug_set_als_variant(0, 0)
