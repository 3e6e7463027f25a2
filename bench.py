"""Benchmark: BASELINE config 1 (standalone CP-ALS truncation) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode fused|sharded|replicas] [--no-cpu] [--no-extra] [--dry-run]

A "step" is one 20-sweep ALS truncation (d=6, Q=256, R=512 -> r=32, lambda=1e-10,
init = first 32 input terms, BASELINE.json configs[1]) of seeded synthetic input.

N = 1 (default):
* ``value``  -- sweeps/s of the fused ALS kernel with inputs resident in HBM,
  CUDA-event timed per step on the launching stream, L2 flushed (256 MiB
  write) between timed steps.
* ``e2e``    -- the same metric through the public API ``cp_approx_als`` with
  pinned HOST buffers: each step copies V and the initial guess host->device
  (double-buffered on a copy stream), runs the truncation and copies the fit back.
* ``roofline`` -- algorithmic fp64 flops of one launch / mean
  launch time vs the measured fp64 DMMA peak (profiles/r01_microbench.txt;
  MEASURED_PEAKS.json has no fp64 entry).
* ``cpu_baseline`` -- the oracle restatement of the reference path (complex128,
  the shipped reference's arithmetic) on this host, 1 BLAS thread and all host
  threads, CPU model from lscpu.
* ``extra_configs`` -- configs 0, 2, 3 (time-steps/s) and 4 (tensors/s) through
  the public API, each with its roofline fraction, a bounded CPU sample, and for
  config 4 an end-to-end figure (host arrays -> packed batch -> hSVD -> host).

N > 1 (``--gpus N`` self-launches N ranks through torch.distributed.run when
WORLD_SIZE is unset; the driver may launch it with torchrun itself): the headline
is BASELINE configs[1] R-SHARDED across the ranks (strong scaling: one truncation,
R/N input terms per GPU, one r x Q right-hand-side all-reduce per mode update);
``extra_configs`` carries config 4 batch-sharded (64/N tensors per GPU, no
communication) and, labelled, independent per-rank replicas of config 1.
NCCL_DEBUG=INFO (subsystem INIT) is set so the communicator init lines of every
rank appear in the log.  The JSON line is printed last, after the process group
is torn down.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
PEAK_SOURCE = "measured fp64 DMMA peak (profiles/r01_microbench.txt); no fp64 entry in MEASURED_PEAKS.json"
WORKLOAD = "cfg1: standalone CP-ALS d=6 Q=256 R=512 r=32, 20 sweeps, lambda=1e-10, init=first 32 terms"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(n: int) -> int:
    """--gpus N without a torchrun environment: start N ranks ourselves (one per GPU)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


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


# --------------------------------------------------------------------------- CPU baselines

def cpu_info() -> dict:
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def _blas_threads(n):
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=n, user_api="blas")


def _timed_loop(fn, seconds, max_n=200):
    n, t0 = 0, time.perf_counter()
    while True:
        fn()
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= max_n:
            return n, el


def cpu_baseline_run(seconds: float = 8.0):
    """Oracle restatement of the reference path (complex128 like the shipped reference,
    fixed lambda + fixed sweeps shims), with 1 BLAS thread and with all host threads."""
    from oracle import cp_als as ocp
    from paper_1803_10270_b200 import workloads
    w = workloads.cfg1(0)
    V = [v.astype(np.complex128) for v in w["V"]]
    init = [u.astype(np.complex128) for u in w["init"]]
    info = cpu_info()
    res = {}
    for th in (1, info["nproc"] or 1):
        with _blas_threads(th):
            ocp.als(V, init, 2, lam=LAM)   # warm-up
            n, el = _timed_loop(lambda: ocp.als(V, init, SWEEPS, lam=LAM), seconds)
        res[th] = (n * SWEEPS / el, n, el)
    best = max(res, key=lambda t: res[t][0])
    v, n, el = res[best]
    return {"value": v, "unit": "sweeps/s", "cores": best, "kind": "port",
            "sample": f"{n} full cfg1 truncations ({n * SWEEPS} sweeps) of the oracle (numpy complex128, "
                      f"reference arithmetic) with {best} BLAS threads, {el:.1f} s wall",
            "cpu_model": info["model"], "nproc": info["nproc"],
            "by_threads": {str(t): round(res[t][0], 2) for t in res}}


def _cfg4_tensor(w, b):
    from oracle import ht_hsvd as oht
    nodes = oht.balanced_tree(w["d"])
    frames, transfers, li, ii = [None] * len(nodes), [None] * len(nodes), 0, 0
    for t, nd in enumerate(nodes):
        if oht.is_leaf(nd):
            frames[t] = w["frames"][b, li]
            li += 1
        else:
            transfers[t] = w["transfers"][b, ii][:, :, :1] if t == 0 else w["transfers"][b, ii]
            ii += 1
    return nodes, frames, transfers


def _cfg4_pool_worker(b):
    from threadpoolctl import threadpool_limits
    from oracle import ht_hsvd as oht
    from paper_1803_10270_b200 import workloads
    with threadpool_limits(limits=1, user_api="blas"):
        w = workloads.cfg4(0, batch=b + 1)
        oht.truncate(_cfg4_tensor(w, b), 16, 0.0)
    return b


def extra_cpu_baselines():
    """Bounded samples of the oracle port (numpy real fp64 -- the reference's complex128
    arithmetic is slower still) for the other BASELINE configs, on the host cores."""
    from oracle import explicit as oex
    from oracle import ht_hsvd as oht
    from oracle import implicit as oim
    from paper_1803_10270_b200 import workloads
    info = cpu_info()
    nproc = info["nproc"] or 1
    out = {}

    def rec(name, value, unit, cores, sample, **kw):
        out[name] = {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": sample,
                     "cpu_model": info["model"], **kw}

    try:
        w = workloads.cfg0(0)
        d = len(w["specs"])
        a = list(-np.asarray(w["a"]))
        mats = [[w["D"] if k == t else None for k in range(d)] for t in range(d)]
        with _blas_threads(1):
            t0 = time.perf_counter()
            oex.run_fused(w["ic"]["factors"], a, mats, w["dt"], w["r"], 100, w["sweeps"], w["lam"])
            el = time.perf_counter() - t0
        rec("cfg0_advection_explicit", 100 / el, "time-steps/s", 1, f"the whole 100-step run, {el:.2f} s "
            "(1 BLAS thread: the 32 x 78 operands are too small to thread)")
        w = workloads.cfg3(0)
        by = {}
        for th in (1, nproc):
            with _blas_threads(th):
                t0 = time.perf_counter()
                oex.run_fused(w["factors"], w["weights"], w["mats"], w["dt"], w["r"], 20, w["sweeps"], w["lam"])
                by[th] = 20 / (time.perf_counter() - t0)
        best = max(by, key=by.get)
        rec("cfg3_bgk_explicit", by[best], "time-steps/s", best, f"20 of 200 fused-AB2 steps, {best} BLAS threads",
            by_threads={str(t): round(v, 2) for t, v in by.items()})
        w = workloads.cfg2(0)
        S, D, a2, dt = w["specs"], w["D"], w["a"], w["dt"]
        d, q = len(S), S[0].Q
        facs = [[None] * d] + [[D if k == t else None for k in range(d)] for t in range(d)]
        tabs = oim.build_tables(facs, [1.0] + [dt * x for x in a2], [1.0] + [0.0] * d, [q] * d)
        with _blas_threads(nproc):
            t0 = time.perf_counter()
            oim.step(w["ic"]["factors"], tabs, 1, w["lam"])
            el = time.perf_counter() - t0
        rec("cfg2_implicit_euler", 1.0 / (el * w["sweeps"]), "time-steps/s", nproc,
            f"1 of the {w['sweeps']} Gauss-Seidel sweeps of one step (direct dense solves, {nproc} BLAS threads), "
            f"scaled; {el:.1f} s")
        # config 4: nproc worker processes x 1 BLAS thread, one tensor each
        import multiprocessing as mpc
        nt = max(2, nproc)
        t0 = time.perf_counter()
        with mpc.get_context("spawn").Pool(nproc) as pool:
            pool.map(_cfg4_pool_worker, range(nt))
        el_pool = time.perf_counter() - t0
        w = workloads.cfg4(0, batch=2)
        with _blas_threads(nproc):
            t0 = time.perf_counter()
            for b in range(2):
                oht.truncate(_cfg4_tensor(w, b), 16, 0.0)
            el_thr = time.perf_counter() - t0
        rec("cfg4_hsvd_batch64", nt / el_pool, "tensors/s", nproc,
            f"{nt} of the 64 tensors on a pool of {nproc} processes x 1 BLAS thread (incl. pool start-up), "
            f"{el_pool:.2f} s", threaded_one_process={"value": 2 / el_thr, "cores": nproc,
                                                      "sample": "2 tensors, one process, threaded BLAS"})
    except Exception as e:  # noqa: BLE001  (a baseline must never break the bench line)
        out["error"] = f"{type(e).__name__}: {e}"
    return out


def run_reference(args):
    """Reference arm: the oracle port of the reference path (complex128 numpy, all host
    BLAS threads), timed on cfg1 with the same steps/warm-up; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
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
    info = cpu_info()
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", info["nproc"] or 1))
    line = {"metric": "CP-ALS sweeps/s", "value": val, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded, seed 0)", "config": {"workload": WORKLOAD, "l2": "n/a (CPU)"},
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "sweeps/s", "cores": cores, "kind": "port",
                             "sample": f"{args.steps} cfg1 truncations of the oracle port (numpy complex128)",
                             "cpu_model": info["model"]},
            "e2e": {"value": val, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- device timing helpers

def _max_over_ranks(ms, world, dev):
    if world == 1:
        return ms
    import torch
    t = torch.tensor([ms], device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def _timed(fn, world, dev, reps=1):
    import torch
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
    return _max_over_ranks(e0.elapsed_time(e1) / reps, world, dev)


def _roof(flops_per_unit, units_per_s):
    tf = flops_per_unit * units_per_s / 1e12
    return {"bound": "tensor", "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": tf / FP64_PEAK_TFLOPS, "flops_per_unit": flops_per_unit}


def cfg0_flops(R=78, r=6, q=32, d=6, sweeps=10, r_in=12):
    """one fused-AB2 step: apply (6 derivative terms on the rank-12 difference), the cross/Gram
    set-up and 10 sweeps of a R -> r truncation (SURVEY 8(d) per-sweep formula)"""
    return (d * 2 * q * q * r_in + d * (2 * r * q * R + 2 * q * r * r)
            + sweeps * d * (4 * r * q * R + 4 * q * r * r + r ** 3 / 3))


def cfg3_flops(n_nonid=66, R=588, r=12, q=64, d=6, sweeps=10, r_in=24):
    """as cfg0 with 24 operator terms (66 non-identity factor applications)"""
    return (n_nonid * 2 * q * q * r_in + d * (2 * r * q * R + 2 * q * r * r)
            + sweeps * d * (4 * r * q * R + 4 * q * r * r + r ** 3 / 3))


def cfg2_circ_flops(q=128, r=16, d=6, ra=7, n_tab=4, sweeps=20):
    """the circulant implicit step: per mode update the DFT of the new
    factor (dense, 8 Q^2 r real flops), its n_tab table Grams by Parseval (8 n_tab Q r^2),
    the Hadamard of the ra^2 term Grams over the other modes (ra^2 d r^2), the assembly of
    Q/2+1 per-frequency Hermitian r x r systems (ra^2 terms, 4 r^2 each) and their
    Cholesky solve + right-hand side (8 (r^3/3 + 2 r^2))"""
    nf = q // 2 + 1
    per = (8 * q * q * r + 8 * n_tab * q * r * r + ra * ra * d * r * r
           + nf * (ra * ra * 4 * r * r + 8 * (r ** 3 / 3 + 2 * r * r)))
    return per * d * sweeps


CFG4_FLOPS = 1.52e9   # QR 207 M + push 404 M + Grams 806 M + eigh 33 M + projection 68 M


def extra_configs(world, rank, dev):
    """Throughput of the other BASELINE configs through the public API (device-resident,
    plus an end-to-end figure for config 4)."""
    import torch
    from paper_1803_10270_b200 import cp, explicit, ht, implicit, operators, workloads
    from paper_1803_10270_b200.basis import BasisSpec
    out = {}

    # config 4: 64 HT tensors, batch-sharded across ranks (no communication)
    w4 = workloads.cfg4(0)
    lo, hi = (64 * rank) // world, (64 * (rank + 1)) // world
    d4, Q4, k4 = w4["d"], w4["Q"], w4["k"]
    specs4 = tuple(BasisSpec(Q4, 1.0, "collocation") for _ in range(d4))
    hF = torch.as_tensor(w4["frames"][lo:hi]).contiguous().pin_memory()
    hB = torch.as_tensor(w4["transfers"][lo:hi]).contiguous().pin_memory()
    batch = ht.HTBatch.from_arrays(specs4, hF, hB)
    res = {"out": None}

    def c4():
        res["out"], _ = ht.truncate_packed(batch, w4["r_max"], w4["eps"], res["out"])
    ms = _timed(c4, world, dev, 3)
    nb = hi - lo
    v4 = 64 / ms * 1e3
    # end to end through the public API: pinned host arrays -> packed device batch ->
    # hSVD -> truncated frames/transfers, ranks and estimates back on the host
    o = res["out"]
    hOF = torch.empty(o.frames.shape, dtype=torch.float64).pin_memory()
    hOB = torch.empty(o.transfers.shape, dtype=torch.float64).pin_memory()
    hE = torch.empty(nb, dtype=torch.float64).pin_memory()

    def e2e4():
        b = ht.HTBatch.from_arrays(specs4, hF, hB, non_blocking=True)
        oo, est = ht.truncate_packed(b, w4["r_max"], w4["eps"])
        hOF.copy_(oo.frames, non_blocking=True)
        hOB.copy_(oo.transfers, non_blocking=True)
        hE.copy_(est, non_blocking=True)
    ms_e2e = _timed(e2e4, world, dev, 3)
    # the reference-shaped call (list of HTTensor in, list out): per-node packing included
    hs = [ht.HTTensor(specs4, ht.balanced_tree(d4), *_cfg4_lists(w4, b)) for b in range(lo, min(hi, lo + 8))]
    ms_list = _timed(lambda: ht.truncate_batch(hs, w4["r_max"], w4["eps"]), world, dev, 1)
    out["cfg4_hsvd_batch64"] = {
        "value": v4, "unit": "tensors/s", "ms_per_batch": ms, "sharding": f"batch {nb} per rank x {world}",
        "roofline": _roof(CFG4_FLOPS, v4),
        "e2e": {"value": 64 / ms_e2e * 1e3, "unit": "tensors/s",
                "h2d_bytes_per_step": int((hF.numel() + hB.numel()) * 8),
                "d2h_bytes_per_step": int((hOF.numel() + hOB.numel() + hE.numel()) * 8),
                "api": "ht.HTBatch.from_arrays + ht.truncate_packed (pinned host arrays, copies in the timed region)"},
        "list_api_tensors_per_s": len(hs) / ms_list * 1e3,
        "list_api": f"ht.truncate_batch on {len(hs)} HTTensor objects (per-node pack/unpack copies included)"}
    del batch, res, hs
    if world > 1:
        return out

    w0 = workloads.cfg0(0)
    L0 = operators.advection_operator(w0["a"], w0["specs"])
    c0 = explicit.ExplicitConfig(dt=w0["dt"], r_max=w0["r"], recipe="fused",
                                 als=cp.ALSApproxConfig(max_sweeps=w0["sweeps"], stall=-np.inf, reg=w0["lam"]))
    f0 = cp.CPTensor(w0["specs"], w0["ic"]["factors"])
    ms = _timed(lambda: explicit.run(f0, L0, c0, w0["steps"]), world, dev)
    v0 = w0["steps"] / ms * 1e3
    out["cfg0_advection_explicit"] = {"value": v0, "unit": "time-steps/s", "ms_per_run_100_steps": ms,
                                      "roofline": _roof(cfg0_flops(), v0),
                                      "note": "latency-bound by construction (SURVEY 8(d)); one CTA per step"}
    w3 = workloads.cfg3(0)
    L3 = operators.SeparableOperator(w3["specs"], tuple(w3["weights"]), tuple(tuple(m) for m in w3["mats"]))
    c3 = explicit.ExplicitConfig(dt=w3["dt"], r_max=w3["r"], recipe="fused",
                                 als=cp.ALSApproxConfig(max_sweeps=w3["sweeps"], stall=-np.inf, reg=w3["lam"]))
    f3 = cp.CPTensor(w3["specs"], w3["factors"])
    ms = _timed(lambda: explicit.run(f3, L3, c3, w3["steps"]), world, dev)
    v3 = w3["steps"] / ms * 1e3
    out["cfg3_bgk_explicit"] = {"value": v3, "unit": "time-steps/s", "ms_per_run_200_steps": ms,
                                "roofline": _roof(cfg3_flops(), v3)}
    w2 = workloads.cfg2(0)
    pair = operators.implicit_euler_pair(operators.advection_operator(w2["a"], w2["specs"]), w2["dt"])
    c2 = implicit.ALSStepConfig(dt=w2["dt"], eps_tol=0.0, max_sweeps=w2["sweeps"], delta_beta=1.0,
                                schedule="gauss-seidel", lam=w2["lam"])
    f2 = cp.CPTensor(w2["specs"], w2["ic"]["factors"])
    steps2 = w2["steps"]
    ws2 = implicit.StepWorkspace(pair, c2)     # operator tables, built once per run (implicit.py:180-210)
    ms = _timed(lambda: implicit.run(f2, pair, c2, steps2, workspace=ws2), world, dev)
    v2 = steps2 / ms * 1e3
    out["cfg2_implicit_euler"] = {"value": v2, "unit": "time-steps/s",
                                  "sample": f"{steps2} steps = the whole run (tables built once per run, outside)",
                                  "ms_per_step": ms / steps2, "roofline": _roof(cfg2_circ_flops(), v2),
                                  "flops_note": "circulant (Fourier block-diagonal) algorithm count, "
                                                "bench.cfg2_circ_flops; the dense direct-solve path the CPU "
                                                "oracle runs costs ~0.4 TFLOP per step (SURVEY 8(d))"}
    return out


def _cfg4_lists(w, b):
    """frames/transfers lists of tensor b in tree order (ht.balanced_tree, ht.py:79-98)"""
    from paper_1803_10270_b200 import ht
    nodes = ht.balanced_tree(w["d"]).nodes
    frames, transfers, li, ii = [None] * len(nodes), [None] * len(nodes), 0, 0
    for t, nd in enumerate(nodes):
        if nd.is_leaf:
            frames[t] = w["frames"][b, li]
            li += 1
        else:
            transfers[t] = w["transfers"][b, ii][:, :, :1] if t == 0 else w["transfers"][b, ii]
            ii += 1
    return frames, transfers


# --------------------------------------------------------------------------- cfg1, one GPU (fused kernel)

def run_fused(args, world, rank, local, dev):
    import torch
    from paper_1803_10270_b200 import cp, workloads
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

    for _ in range(args.warmup):
        U.copy_(I0.data)
        cp._als_device(T, U, RANK_R, cfg, None, info)
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
    cp._check_info(info)
    per = [e0.elapsed_time(e1) for e0, e1 in evs]
    tot_ms = _max_over_ranks(sum(per), world, dev)
    value = world * args.steps * SWEEPS / (tot_ms / 1e3)
    ms_per_step = tot_ms / args.steps
    achieved_tf = FLOPS_PER_STEP / (ms_per_step / 1e3) / 1e12

    # steady-state sweeps/s without setup: 10- vs 20-sweep truncations
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

    # ---- e2e: public API with pinned host buffers, H2D + call + D2H every step
    # (double-buffered: step i+1's inputs cross on a copy stream while step i computes)
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
            o = cp.cp_approx_als(Tt, RANK_R, cfg, init=It, sync=False)
            consumed[b].record(stream)
            # the fit's device->host read on the copy stream, overlapping the next truncation
            with torch.cuda.stream(s_copy):
                s_copy.wait_event(consumed[b])
                hOut.copy_(o.data, non_blocking=True)
            outs.append(o)

    e2e_run(max(2, args.warmup))
    torch.cuda.synchronize()
    e2e_samples = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_run(args.steps)
        stream.wait_stream(s_copy)   # the last device->host read is inside the timed region
        e1.record(stream)
        torch.cuda.synchronize()
        for o in outs:       # deferred status checks (ConditioningError would raise here)
            cp.check(o)
        outs.clear()
        e2e_samples.append(e0.elapsed_time(e1))
    e2e_ms = _max_over_ranks(sorted(e2e_samples)[1], world, dev)
    e2e_val = world * args.steps * SWEEPS / (e2e_ms / 1e3)
    traffic, traffic_src = None, None
    for name in ("r02_als_ncu.json", "r01_als_ncu.json"):
        prof_json = ROOT / "profiles" / name
        if prof_json.exists():
            try:
                pj = json.loads(prof_json.read_text())
                traffic, traffic_src = pj.get("dram_bytes_per_launch"), pj.get("source")
                break
            except Exception:
                traffic = None
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
                     "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": (f"tp::als_w ({plan['ctas']} CTAs, {plan['smem_bytes']} B smem; a step = one batched bgemm "
                                "launch (W_k = V_k^T V_k) + als_w + the als_rows fallback "
                                "launch that returns at once; achieved = reference-algorithm flops / whole step)")
                               if plan["kernel"] == "als_w" else
                               f"tp::{plan['kernel']}<32> (one launch per step; {plan['ctas']} CTAs, "
                               f"cluster {plan['cluster']}, {plan['smem_bytes']} B smem)",
                     "flops_per_launch": FLOPS_PER_STEP, "peak_source": PEAK_SOURCE},
        "gpu_launches": args.steps * (3 if plan["kernel"] == "als_w" else 1),
        "clocks": clk.summary(),
        "wall_s_timed_region": t_wall,
        "steady_state_sweeps_per_s": steady,
        "setup_ms": (2 * ms10 - ms20) if steady else None,
    }
    return line


# --------------------------------------------------------------------------- cfg1 R-sharded (N > 1 headline)

def run_sharded(args, world, rank, local, dev):
    """One config-1 truncation R-sharded across the ranks (strong scaling): rank g holds
    input terms [R g/N, R (g+1)/N) and the replicated guess; per mode update one r x Q
    right-hand-side exchange (parallel.ShardedALS)."""
    import torch
    from paper_1803_10270_b200 import cp, parallel, workloads
    w = workloads.cfg1(seed=0)
    lo, hi = parallel.shard_range(R, world, rank)
    specs = w["specs"]
    Vs = cp.CPTensor(specs, [v[:, lo:hi] for v in w["V"]])
    I0 = cp.CPTensor(specs, w["init"])
    cfg = cp.ALSApproxConfig(max_sweeps=SWEEPS, tol=0.0, stall=-np.inf, reg=LAM)
    drv = parallel.make_sharded_als(Vs, RANK_R, cfg)
    stream = torch.cuda.current_stream(dev)
    U = I0.data.clone()
    drv.prepare(U)

    def one():
        U.copy_(I0.data)
        drv.run(U)

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
    drv.check()
    tot_ms = _max_over_ranks(e0.elapsed_time(e1), world, dev)
    ms_per_step = tot_ms / args.steps
    value = args.steps * SWEEPS / (tot_ms / 1e3)
    # e2e through the public sharded API: this rank's slab + the guess from pinned host
    # memory, the truncation, the (replicated) fit back to the host
    hV = torch.cat([torch.as_tensor(np.ascontiguousarray(v[:, lo:hi])).reshape(-1) for v in w["V"]]).pin_memory()
    hI = torch.cat([torch.as_tensor(u).reshape(-1) for u in w["init"]]).pin_memory()
    hOut = torch.empty_like(hI).pin_memory()

    def e2e_one():
        Vd = cp.CPTensor(specs, data=hV.to(dev, non_blocking=True), rank=hi - lo)
        Id = cp.CPTensor(specs, data=hI.to(dev, non_blocking=True), rank=RANK_R)
        o = parallel.sharded_cp_approx_als(Vd, Id, cfg, check=False)
        hOut.copy_(o.data, non_blocking=True)
    e2e_one()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_one()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = _max_over_ranks(e0.elapsed_time(e1), world, dev)
    achieved_tf = FLOPS_PER_STEP / (ms_per_step / 1e3) / 1e12
    line = {"metric": "CP-ALS sweeps/s", "value": value, "unit": "sweeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, seed 0)",
            "config": {"workload": WORKLOAD, "parallelism": f"R-sharded x{world} ({drv.describe()})",
                       "l2": "inputs L2-resident, not flushed (the slab is re-read every mode update)"},
            "e2e": {"value": args.steps * SWEEPS / (e2e_ms / 1e3), "unit": "sweeps/s",
                    "h2d_bytes_per_step": int((hV.numel() + hI.numel()) * 8),
                    "d2h_bytes_per_step": int(hOut.numel() * 8),
                    "api": "parallel.sharded_cp_approx_als (per-rank slab + guess H2D, fit D2H)"},
            "roofline": {"bound": "tensor", "achieved": achieved_tf / world, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved_tf / world / FP64_PEAK_TFLOPS, "traffic": None,
                         "kernel": drv.kernel_name(), "flops_per_launch": FLOPS_PER_STEP / world,
                         "peak_source": PEAK_SOURCE},
            "gpu_launches": args.steps * drv.launches_per_truncation(), "clocks": clk.summary()}
    return line


def run_dry(args):
    """--dry-run: the launcher / rank / max-over-ranks plumbing on CPU (gloo), no kernels."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    buf = torch.zeros(RANK_R * Q, dtype=torch.float64)   # the r x Q exchange of one mode update
    t0 = time.perf_counter()
    for _ in range(args.steps * D):
        if world > 1:
            dist.all_reduce(buf)
    ms = (time.perf_counter() - t0) * 1e3
    if world > 1:
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": "CP-ALS sweeps/s", "value": None, "unit": "sweeps/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1),
                          "dry_run": True, "config": {"workload": WORKLOAD, "backend": "gloo (CPU)"}}), flush=True)


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    mode = args.mode or ("fused" if world == 1 else "sharded")
    if mode == "sharded":
        line = run_sharded(args, world, rank, local, dev)
        if not args.no_extra:
            rep = run_fused(args, world, rank, local, dev)      # labelled extra: independent replicas
            line["extra_configs"] = {"cfg1_replicas_weak": {"value": rep["value"], "unit": "sweeps/s",
                                                            "note": "independent cfg1 truncation per rank "
                                                                    "(weak scaling), not the headline"}}
    else:
        line = run_fused(args, world, rank, local, dev)
        if world == 1 and not args.no_cpu and rank == 0:
            line["cpu_baseline"] = cpu_baseline_run(args.cpu_seconds)
    if not args.no_extra:
        extras = extra_configs(world, rank, dev)
        if rank == 0 and world == 1 and not args.no_cpu:
            for name, cb in extra_cpu_baselines().items():
                if name in extras:
                    extras[name]["cpu_baseline"] = cb
        line.setdefault("extra_configs", {}).update(extras)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--mode", choices=["fused", "sharded", "replicas"], default=None)
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--dry-run", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.mode == "replicas":
        args.mode = "fused"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
