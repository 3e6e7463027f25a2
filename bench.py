"""Benchmark: BASELINE config 1 (standalone CP-ALS truncation) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--grid P]

A "step" is one 20-sweep ALS truncation (d=6, Q=256, R=512 -> r=32, lambda=1e-10,
init = first 32 input terms, BASELINE.json configs[1]) of seeded synthetic input.

* ``value``  -- sweeps/s of the fused ALS kernel with inputs resident in HBM,
  CUDA-event timed per step on the launching stream, L2 flushed (256 MiB
  write) between timed steps; whole-job aggregate over ranks (max time).
* ``e2e``    -- the same metric through the public API ``cp_approx_als`` with
  pinned HOST buffers: each step copies V and the initial guess host->device
  (double-buffered on a copy stream, overlapping the previous step), runs the
  truncation (incl. its one-int status check) and copies the fit back.
* ``roofline`` -- algorithmic fp64 flops of one launch / mean
  launch time vs the measured fp64 DMMA peak (profiles/r01_microbench.txt;
  MEASURED_PEAKS.json has no fp64 entry).
* ``cpu_baseline`` -- the oracle restatement of the reference path (complex128,
  like the shipped reference) timed on this host's cores on a bounded sample.

N > 1 (torchrun): ``--mode replicas`` (default for N > 1) runs an independent
config-1 truncation per rank (weak scaling: batches of independent truncations
sharded with no communication); ``--mode sharded`` shards the R input terms of ONE
truncation across ranks with an NCCL all-reduce of the r x Q right-hand side per
mode update (strong scaling, BASELINE configs[1]) -- latency-bound at this size
(120 dependent all-reduces per 1.5 ms truncation), see DESIGN.md section 7.
``extra_configs`` reports device-resident throughput of configs 0, 2, 3 (rank 0,
N = 1) and of config 4 (batch of 64 HT tensors sharded across ranks), each with a
bounded ``cpu_baseline`` sample of the oracle port on the host cores (N = 1).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

D, Q, R, RANK_R, SWEEPS, LAM = 6, 256, 512, 32, 20, 1e-10
# algorithmic flops (FMA = 2, no symmetry savings), SURVEY 8(d):
SWEEP_FLOPS = D * (4 * RANK_R * Q * R + 4 * Q * RANK_R ** 2 + RANK_R ** 3 / 3)      # 107.0 MFLOP
SETUP_FLOPS = D * 2 * RANK_R * Q * R + D * 2 * Q * RANK_R ** 2                       # crosses + Grams
# the target self-norm (805 MFLOP) only runs when a trace / stopping rule needs it; off here
FLOPS_PER_STEP = SWEEPS * SWEEP_FLOPS + SETUP_FLOPS
FP64_PEAK_TFLOPS = 37.08   # measured DMMA m8n8k4 f64 on this pool's B200 (profiles/r01_microbench.txt)
WORKLOAD = "cfg1: standalone CP-ALS d=6 Q=256 R=512 r=32, 20 sweeps, lambda=1e-10, init=first 32 terms"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline_run(seconds: float = 12.0):
    """Oracle restatement of the reference path (complex128 like the shipped reference,
    fixed lambda + fixed sweeps shims), all host threads via OpenBLAS."""
    from oracle import cp_als as ocp
    from paper_1803_10270_b200 import workloads
    w = workloads.cfg1(0)
    V = [v.astype(np.complex128) for v in w["V"]]
    init = [u.astype(np.complex128) for u in w["init"]]
    ocp.als(V, init, 2, lam=LAM)   # warm-up
    n, t0 = 0, time.perf_counter()
    while True:
        ocp.als(V, init, SWEEPS, lam=LAM)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 200:
            break
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    return {"value": n * SWEEPS / el, "unit": "sweeps/s", "cores": cores, "kind": "port",
            "sample": f"{n} full cfg1 truncations ({n * SWEEPS} sweeps) of the oracle (numpy complex128, "
                      f"reference arithmetic), {el:.1f} s wall"}


def extra_cpu_baselines():
    """Bounded samples of the oracle port (numpy, real fp64 -- the reference's complex128
    arithmetic is slower still) for the other BASELINE configs, on the host cores."""
    from oracle import explicit as oex
    from oracle import ht_hsvd as oht
    from oracle import implicit as oim
    from paper_1803_10270_b200 import workloads
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    out = {}

    def rec(name, value, unit, sample):
        out[name] = {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": sample}

    try:
        w = workloads.cfg0(0)
        d = len(w["specs"])
        a = list(-np.asarray(w["a"]))
        mats = [[w["D"] if k == t else None for k in range(d)] for t in range(d)]
        t0 = time.perf_counter()
        oex.run_fused(w["ic"]["factors"], a, mats, w["dt"], w["r"], 100, w["sweeps"], w["lam"])
        el = time.perf_counter() - t0
        rec("cfg0_advection_explicit", 100 / el, "time-steps/s", f"the whole 100-step run, {el:.2f} s")
        w = workloads.cfg3(0)
        t0 = time.perf_counter()
        oex.run_fused(w["factors"], w["weights"], w["mats"], w["dt"], w["r"], 30, w["sweeps"], w["lam"])
        el = time.perf_counter() - t0
        rec("cfg3_bgk_explicit", 30 / el, "time-steps/s", f"30 of 200 fused-AB2 steps, {el:.2f} s")
        w = workloads.cfg2(0)
        S, D, a2, dt = w["specs"], w["D"], w["a"], w["dt"]
        d, q = len(S), S[0].Q
        facs = [[None] * d] + [[D if k == t else None for k in range(d)] for t in range(d)]
        tabs = oim.build_tables(facs, [1.0] + [dt * x for x in a2], [1.0] + [0.0] * d, [q] * d)
        t0 = time.perf_counter()
        oim.step(w["ic"]["factors"], tabs, 1, w["lam"])
        el = time.perf_counter() - t0
        rec("cfg2_implicit_euler", 1.0 / (el * w["sweeps"]), "time-steps/s",
            f"1 of the {w['sweeps']} Gauss-Seidel sweeps of one step (direct dense solves), scaled; {el:.1f} s")
        w = workloads.cfg4(0, batch=2)
        nodes = oht.balanced_tree(w["d"])
        t0 = time.perf_counter()
        for b in range(2):
            frames, transfers, li, ii = [None] * len(nodes), [None] * len(nodes), 0, 0
            for t, nd in enumerate(nodes):
                if oht.is_leaf(nd):
                    frames[t] = w["frames"][b, li]; li += 1
                else:
                    transfers[t] = w["transfers"][b, ii][:, :, :1] if t == 0 else w["transfers"][b, ii]; ii += 1
            oht.truncate((nodes, frames, transfers), 16, 0.0)
        el = time.perf_counter() - t0
        rec("cfg4_hsvd_batch64", 2 / el, "tensors/s", f"2 of the 64 tensors (one process, threaded BLAS), {el:.2f} s")
    except Exception as e:  # noqa: BLE001  (a baseline must never break the bench line)
        out["error"] = f"{type(e).__name__}: {e}"
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    for _ in range(args.warmup):
        pass
    from oracle import cp_als as ocp
    from paper_1803_10270_b200 import workloads
    w = workloads.cfg1(0)
    V = [v.astype(np.complex128) for v in w["V"]]
    init = [u.astype(np.complex128) for u in w["init"]]
    for _ in range(max(args.warmup, 1)):
        ocp.als(V, init, 2, lam=LAM)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ocp.als(V, init, SWEEPS, lam=LAM)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = args.steps * SWEEPS / tot
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    line = {"metric": "CP-ALS sweeps/s", "value": val, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, seed 0)",
            "config": {"workload": WORKLOAD, "l2": "n/a (CPU)"}, "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": cores, "kind": "port",
                             "sample": f"{args.steps} cfg1 truncations of the oracle port (numpy complex128)"},
            "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def extra_configs(world, rank, dev):
    """Device-resident throughput of the other BASELINE configs through the public API."""
    import torch
    from paper_1803_10270_b200 import cp, explicit, ht, implicit, operators, workloads
    out = {}

    def timed(fn, reps=1):
        fn()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # config 4: 64 HT tensors, batch-sharded across ranks (no communication)
    w4 = workloads.cfg4(0)
    lo, hi = (64 * rank) // world, (64 * (rank + 1)) // world
    from paper_1803_10270_b200 import _lib
    F = torch.as_tensor(w4["frames"][lo:hi]).to(dev)
    B = torch.as_tensor(w4["transfers"][lo:hi]).to(dev)
    nb, d, Q, k, ro = hi - lo, w4["d"], w4["Q"], w4["k"], 16
    OF = torch.zeros((nb, d, Q, ro), dtype=torch.float64, device=dev)
    OB = torch.zeros((nb, d - 1, ro, ro, ro), dtype=torch.float64, device=dev)
    rk = torch.zeros((nb, 2 * d - 1), dtype=torch.int32, device=dev)
    est = torch.zeros(nb, dtype=torch.float64, device=dev)
    nrm = torch.zeros(nb, dtype=torch.float64, device=dev)
    L = _lib.lib()
    ws = torch.empty(L.tp_ht_truncate_ws_bytes(d, Q, k, nb), dtype=torch.uint8, device=dev)

    def c4():
        _lib.check(L.tp_ht_truncate_f64(d, Q, k, nb, F.data_ptr(), B.data_ptr(), ro, 0.0, OF.data_ptr(),
                                        OB.data_ptr(), rk.data_ptr(), est.data_ptr(), nrm.data_ptr(), ws.data_ptr(),
                                        ws.numel(), _lib.stream_ptr(dev)))
    ms = timed(c4, 3)
    out["cfg4_hsvd_batch64"] = {"value": 64 / ms * 1e3, "unit": "tensors/s", "ms_per_batch": ms,
                                "flops_per_tensor": 1.52e9, "achieved_tflops": 64 * 1.52e9 / (ms * 1e-3) / 1e12,
                                "sharding": f"batch {nb} per rank"}
    del F, B, OF, OB, ws
    if world > 1:
        return out
    w0 = workloads.cfg0(0)
    L0 = operators.advection_operator(w0["a"], w0["specs"])
    c0 = explicit.ExplicitConfig(dt=w0["dt"], r_max=w0["r"], recipe="fused",
                                 als=cp.ALSApproxConfig(max_sweeps=w0["sweeps"], stall=-np.inf, reg=w0["lam"]))
    f0 = cp.CPTensor(w0["specs"], w0["ic"]["factors"])
    ms = timed(lambda: explicit.run(f0, L0, c0, w0["steps"]))
    out["cfg0_advection_explicit"] = {"value": w0["steps"] / ms * 1e3, "unit": "time-steps/s",
                                      "ms_per_run_100_steps": ms}
    w3 = workloads.cfg3(0)
    L3 = operators.SeparableOperator(w3["specs"], tuple(w3["weights"]), tuple(tuple(m) for m in w3["mats"]))
    c3 = explicit.ExplicitConfig(dt=w3["dt"], r_max=w3["r"], recipe="fused",
                                 als=cp.ALSApproxConfig(max_sweeps=w3["sweeps"], stall=-np.inf, reg=w3["lam"]))
    f3 = cp.CPTensor(w3["specs"], w3["factors"])
    ms = timed(lambda: explicit.run(f3, L3, c3, w3["steps"]))
    out["cfg3_bgk_explicit"] = {"value": w3["steps"] / ms * 1e3, "unit": "time-steps/s",
                                "ms_per_run_200_steps": ms}
    w2 = workloads.cfg2(0)
    pair = operators.implicit_euler_pair(operators.advection_operator(w2["a"], w2["specs"]), w2["dt"])
    c2 = implicit.ALSStepConfig(dt=w2["dt"], eps_tol=0.0, max_sweeps=w2["sweeps"], delta_beta=1.0,
                                schedule="gauss-seidel", lam=w2["lam"])
    f2 = cp.CPTensor(w2["specs"], w2["ic"]["factors"])
    steps2 = w2["steps"]
    ws2 = implicit.StepWorkspace(pair, c2)     # operator tables, built once per run (implicit.py:180-210)
    ms = timed(lambda: implicit.run(f2, pair, c2, steps2, workspace=ws2))
    out["cfg2_implicit_euler"] = {"value": steps2 / ms * 1e3, "unit": "time-steps/s",
                                  "sample": f"{steps2} steps = the whole run (tables built once per run, outside)",
                                  "ms_per_step": ms / steps2}
    _ = ht
    return out


def run_sharded(args, world, rank, local, dev):
    """One config-1 truncation R-sharded across ranks (strong scaling)."""
    import torch
    from paper_1803_10270_b200 import cp, parallel, workloads
    w = workloads.cfg1(seed=0)
    lo, hi = parallel.shard_range(R, world, rank)
    specs = w["specs"]
    Vs = cp.CPTensor(specs, [v[:, lo:hi] for v in w["V"]])
    I0 = cp.CPTensor(specs, w["init"])
    cfg = cp.ALSApproxConfig(max_sweeps=SWEEPS, tol=0.0, stall=-np.inf, reg=LAM)
    comm = parallel.TorchDistComm() if world > 1 else parallel.LocalComm()
    ops = parallel.DeviceShardOps(Vs, RANK_R)
    U = I0.data.clone()
    drv = parallel.ShardedALS(ops, comm, cfg)
    stream = torch.cuda.current_stream(dev)
    U.copy_(I0.data)
    drv.capture(U, D)      # whole truncation (2520 launches incl. 120 all-reduces) as one CUDA graph

    def one():
        U.copy_(I0.data)
        drv.replay()

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            one()
        e1.record(stream)
        torch.cuda.synchronize()
    ops.check()
    tot_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    return tot_ms, clk.summary()


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mode = args.mode or "fused"     # N > 1: independent truncation per rank (replicas)
    if mode == "sharded":
        dev = torch.device("cuda", local)
        tot_ms, clocks = run_sharded(args, world, rank, local, dev)
        ms_per_step = tot_ms / args.steps
        value = args.steps * SWEEPS / (tot_ms / 1e3)
        extras = extra_configs(world, rank, dev) if not args.no_extra else {}
        if rank == 0:
            achieved_tf = FLOPS_PER_STEP / (ms_per_step / 1e3) / 1e12
            line = {"metric": "CP-ALS sweeps/s", "value": value, "unit": "sweeps/s", "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                    "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, seed 0)",
                    "config": {"workload": WORKLOAD, "parallelism": f"R-sharded x{world} (NCCL all-reduce of the "
                                                                   f"r x Q rhs per mode update)",
                               "l2": "inputs L2-resident, not flushed (host-orchestrated mode steps)"},
                    "roofline": {"bound": "tensor", "achieved": achieved_tf / world, "peak": FP64_PEAK_TFLOPS,
                                 "unit": "TFLOP/s", "frac": achieved_tf / world / FP64_PEAK_TFLOPS, "traffic": None,
                                 "kernel": "tp_als_shard_* mode steps (per GPU)"},
                    "gpu_launches": args.steps * (SWEEPS * D * 6 + 2 * D), "clocks": clocks,
                    "extra_configs": extras}
            print(json.dumps(line), flush=True)
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    from paper_1803_10270_b200 import cp, workloads
    from paper_1803_10270_b200 import _lib
    dev = torch.device("cuda", local)
    plan = cp.als_plan([Q] * D, R, RANK_R, args.grid)
    w = workloads.cfg1(seed=rank)
    specs = w["specs"]
    T = cp.CPTensor(specs, w["V"])
    I0 = cp.CPTensor(specs, w["init"])
    cfg = cp.ALSApproxConfig(max_sweeps=SWEEPS, tol=0.0, stall=-np.inf, reg=LAM, grid=args.grid)
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    U = I0.data.clone()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def one():
        U.copy_(I0.data)
        cp._als_device(T, U, RANK_R, cfg, None, info)

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for e0, e1 in evs:
            flush.fill_(1.0)               # L2 flush outside the timed interval
            U.copy_(I0.data)
            e0.record(stream)
            cp._als_device(T, U, RANK_R, cfg, None, info)
            e1.record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    _ = cp._check_info(info)
    per = [e0.elapsed_time(e1) for e0, e1 in evs]
    tot_ms = sum(per)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = world * args.steps * SWEEPS / (tot_ms / 1e3)
    ms_per_step = tot_ms / args.steps
    achieved_tf = FLOPS_PER_STEP / (ms_per_step / 1e3) / 1e12

    # steady-state sweeps/s without setup: the same truncation with 10
    # and with 20 sweeps, per-sweep time = difference / 10 (outside the timed K steps)
    def t_sweeps(n_sw, reps=5):
        c = cp.ALSApproxConfig(max_sweeps=n_sw, tol=0.0, stall=-np.inf, reg=LAM, grid=args.grid)
        tt = 0.0
        for _ in range(reps):
            flush.fill_(1.0)
            U.copy_(I0.data)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            cp._als_device(T, U, RANK_R, c, None, info)
            a1.record(stream)
            torch.cuda.synchronize()
            tt += a0.elapsed_time(a1)
        return tt / reps
    ms10, ms20 = t_sweeps(10), t_sweeps(20)
    steady = 10.0 / ((ms20 - ms10) / 1e3) if ms20 > ms10 else None

    # ---- e2e: public API with pinned host buffers, H2D + call + D2H every step.
    # Two device buffer sets: the host->device copy of step i+1 runs on a copy
    # stream while step i computes (the production pipeline); every step's inputs
    # still cross PCIe/C2C inside the timed region and its fit is read back.
    hV = torch.cat([torch.as_tensor(v).reshape(-1) for v in w["V"]]).pin_memory()
    hI = torch.cat([torch.as_tensor(u).reshape(-1) for u in w["init"]]).pin_memory()
    hOut = torch.empty_like(hI).pin_memory()
    dV = [torch.empty_like(hV, device=dev) for _ in range(2)]
    dI = [torch.empty_like(hI, device=dev) for _ in range(2)]
    s_copy = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def issue_copy(b):
        with torch.cuda.stream(s_copy):
            s_copy.wait_event(consumed[b])
            dV[b].copy_(hV, non_blocking=True)
            dI[b].copy_(hI, non_blocking=True)
            copied[b].record(s_copy)

    outs = []

    def e2e_run(n):
        for b in range(2):
            consumed[b].record(stream)
        issue_copy(0)
        for i in range(n):
            b = i & 1
            if i + 1 < n:
                issue_copy(b ^ 1)
            stream.wait_event(copied[b])
            Tt = cp.CPTensor(specs, data=dV[b], rank=R)
            It = cp.CPTensor(specs, data=dI[b], rank=RANK_R)
            out = cp.cp_approx_als(Tt, RANK_R, cfg, init=It, sync=False)
            consumed[b].record(stream)
            hOut.copy_(out.data, non_blocking=True)
            outs.append(out)

    e2e_run(max(2, args.warmup))
    torch.cuda.synchronize()
    # three timed repetitions of the K steps (host-side copy throughput varies
    # run to run on a shared box); the median is reported, all three are kept
    e2e_samples = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_run(args.steps)
        s_copy.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        for o in outs:       # deferred status checks (ConditioningError would raise here)
            cp.check(o)
        outs.clear()
        e2e_samples.append(e0.elapsed_time(e1))
    e2e_ms = sorted(e2e_samples)[1]
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = world * args.steps * SWEEPS / (e2e_ms / 1e3)
    traffic = None
    prof_json = ROOT / "profiles" / "r01_als_ncu.json"
    if prof_json.exists():
        try:
            traffic = json.loads(prof_json.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": "CP-ALS sweeps/s", "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded N(0,1)/sqrt(Q), seed = rank)",
            "config": {"workload": WORKLOAD, "l2": "flushed (256 MiB write) between timed steps",
                       "grid_ctas": plan["ctas"], "cluster_ctas": plan["cluster"],
                       "target_norm": "not computed (no trace / stopping rule)",
                       "multi_gpu": "independent replicas per rank (weak)" if world > 1 else "single GPU"},
            "e2e": {"value": e2e_val, "unit": "sweeps/s", "h2d_bytes_per_step": int((hV.numel() + hI.numel()) * 8),
                    "d2h_bytes_per_step": int(hOut.numel() * 8 + 8),
                    "samples_sweeps_per_s": [world * args.steps * SWEEPS / (m / 1e3) for m in e2e_samples],
                    "statistic": "median of 3 timed repetitions of the K steps"},
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "kernel": f"tp::{plan['kernel']}<32> (one launch per step; {plan['ctas']} CTAs, "
                                   f"cluster {plan['cluster']}, {plan['smem_bytes']} B smem)",
                         "flops_per_launch": FLOPS_PER_STEP,
                         "peak_source": "measured fp64 DMMA peak (profiles/r01_microbench.txt); no fp64 entry in "
                                        "MEASURED_PEAKS.json"},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "wall_s_timed_region": t_wall,
            "steady_state_sweeps_per_s": steady,
            "setup_ms": (2 * ms10 - ms20) if steady else None,
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_run(args.cpu_seconds)
    extras = extra_configs(world, rank, dev) if not args.no_extra else {}
    if rank == 0 and world == 1 and not args.no_cpu and not args.no_extra:
        for name, cb in extra_cpu_baselines().items():
            if name in extras:
                extras[name]["cpu_baseline"] = cb
    if rank == 0:
        line["extra_configs"] = extras
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    _ = _lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--mode", choices=["fused", "sharded", "replicas"], default=None)   # replicas == fused per rank
    ap.add_argument("--no-extra", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
