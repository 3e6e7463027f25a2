"""Cluster-row ALS kernel (variant 8): parity vs the oracle / other variants, timing, phases."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp, workloads  # noqa: E402
from oracle import cp_als as ocp, metrics  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
L.tp_debug_set_als_rows.argtypes = [ctypes.c_int, ctypes.c_int]
L.tp_cp_als_plan.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                             ctypes.POINTER(ctypes.c_int)]


def plan(qs, R, r):
    q = (ctypes.c_int * len(qs))(*qs)
    out = (ctypes.c_int * 4)()
    st = L.tp_cp_als_plan(len(qs), q, R, r, 0, out)
    return st, list(out)


# small parity cases first (oracle)
rng = np.random.default_rng(1)
for (qs, R, r, sw) in [((32, 32, 32), 96, 8, 5), ((48, 40, 64, 36), 200, 16, 6), ((64,) * 5, 300, 30, 4),
                       ((256,) * 3, 130, 32, 3), ((20, 33, 17, 40), 64, 12, 5)]:
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    from paper_1803_10270_b200.basis import BasisSpec
    S = tuple(BasisSpec(q, 1.0, "collocation") for q in qs)
    ref = ocp.als(V, init, sw, lam=1e-10)
    L.tp_debug_set_als_variant(8, 0)
    st, pl = plan(qs, R, r)
    try:
        out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=sw, stall=-np.inf, reg=1e-10),
                               init=cp.CPTensor(S, init))
        rel = metrics.cp_rel_diff(ref, out.to_numpy())
        print("parity", qs, R, r, "plan", st, pl, "rel %.3e" % rel, flush=True)
    except Exception as e:  # noqa: BLE001
        print("parity", qs, R, r, "plan", st, pl, "FAILED", e, flush=True)
    L.tp_debug_set_als_variant(0, 0)

w = workloads.cfg1(0)
T = cp.CPTensor(w["specs"], w["V"])
I0 = cp.CPTensor(w["specs"], w["init"])
info = torch.zeros(2, dtype=torch.int32, device=T.data.device)
cfg = cp.ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
U = I0.data.clone()
outs = {}
ref = ocp.als([np.asarray(v) for v in w["V"]], [np.asarray(v) for v in w["init"]], 20, lam=1e-10)
L.tp_debug_set_als_rows_mc.argtypes = [ctypes.c_int]
for name, var, cs, pr in [("rows16", 8, 16, 0), ("unsplit", 8, 16, 0)]:
    L.tp_debug_set_als_rows_mc(0 if pr == -2 else 1)
    L.tp_debug_set_als_rows_split.argtypes = [ctypes.c_int]
    L.tp_debug_set_als_rows_split(0 if name == "unsplit" else 1)
    pr = max(pr, 0)
    L.tp_debug_set_als_variant(var, cs)
    L.tp_debug_set_als_rows(1 if var == 8 else 0, pr)
    st, pl = plan([256] * 6, 512, 32)
    try:
        for _ in range(2):
            U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(name, "plan", st, pl, "failed:", e, flush=True)
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    outs[name] = cp.CPTensor(w["specs"], data=U.clone(), rank=32).to_numpy()
    rel = metrics.cp_rel_diff(ref, outs[name])
    print(f"{name:9s} plan {pl} {ms*1e3:8.1f} us/truncation {20/ms*1e3:8.0f} sweeps/s  info={info.tolist()}  "
          f"rel vs oracle {rel:.2e}", flush=True)
    if var == 8:
        prof = torch.zeros(16, dtype=torch.int64, device="cuda")
        L.tp_debug_set_als_profile.argtypes = [ctypes.c_void_p]
        L.tp_debug_set_als_profile(prof.data_ptr())
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
        torch.cuda.synchronize()
        L.tp_debug_set_als_profile(None)
        p = prof.cpu().numpy() / 120.0
        lab = {7: "Y dmma", 8: "slot store", 1: "signal", 2: "inverse", 3: "wait", 4: "gather", 5: "solve",
               9: "xch dmma+push", 10: "B1", 11: "reduce+publish", 6: "B2", 0: "loop", 12: "owner sums", 13: "H blocks", 14: "xch dmma", 15: "A blk"}
        print("   cycles per mode update: " + " | ".join("%s %.0f" % (lab[i], p[i]) for i in
                                                          (7, 8, 1, 2, 3, 4, 5, 14, 9, 10, 12, 15, 13, 11, 6, 0)), flush=True)
    if var == 8:
        L.tp_debug_set_als_ns.argtypes = [ctypes.c_int]
        L.tp_debug_set_als_ns(0)
        U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info); torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            U.copy_(I0.data); cp._als_device(T, U, 32, cfg, None, info)
        e1.record(); torch.cuda.synchronize()
        L.tp_debug_set_als_ns(6)
        rel = metrics.cp_rel_diff(ref, cp.CPTensor(w["specs"], data=U.clone(), rank=32).to_numpy())
        print(f"   exact-inverse-only: {e0.elapsed_time(e1) / 3 * 1e3:8.1f} us/truncation rel vs oracle {rel:.2e}", flush=True)
# trace / stopping path: rows vs cluster variant
for var, cs in [(2, 4), (8, 16)]:
    L.tp_debug_set_als_variant(var, cs)
    L.tp_debug_set_als_rows(1 if var == 8 else 0, 0)
    tr = []
    out = cp.cp_approx_als(T, 32, cp.ALSApproxConfig(max_sweeps=8, stall=-np.inf, reg=1e-10), init=I0, trace=tr)
    out2 = cp.cp_approx_als(T, 32, cp.ALSApproxConfig(max_sweeps=50, tol=0.0, stall=1e-3, reg=1e-10), init=I0, trace=(tr2 := []))
    print("variant", var, "trace", ["%.12e" % t for t in tr[:3]], "...", "%.12e" % tr[-1], " stall-stop sweeps", len(tr2), flush=True)
L.tp_debug_set_als_variant(0, 0)
L.tp_debug_set_als_rows(1, 0)
L.tp_debug_set_als_rows_mc(1)
