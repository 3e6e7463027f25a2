"""Multi-GPU partitioning of the hot path.

* Config 1 -- input-rank (R) sharding of one CP-ALS truncation: rank g owns a
  contiguous block of the R target terms; every mode update needs ONE exchange,
  the sum of the r x Q right-hand-side partials (64 KiB at config 1), done with
  ``torch.distributed.all_reduce`` (NCCL over NVLink on B200, gloo on CPU).  The
  r x r Grams and the guess are replicated, so the solve is redundant and no
  other communication is needed.  Results equal the single-device
  ``cp_approx_als`` up to summation order.
* Config 4 -- batch sharding: independent HT truncations, no communication.

The per-shard arithmetic is behind a small ``ops`` interface (``DeviceShardOps``
= the sm_100a C-ABI kernels); ``ShardedALS`` only orchestrates, so the same host
logic is exercised by multi-process gloo tests on CPU.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .cp import ALSApproxConfig, CPTensor

__all__ = ["shard_range", "ShardedALS", "DeviceShardOps", "TorchDistComm", "LocalComm", "shard_batch",
           "FusedShardedALS", "GraphShardedALS", "make_sharded_als", "sharded_cp_approx_als", "simulate_sharded_als"]


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block partition [lo, hi) of n items (same split as the kernels' CTA slabs)."""
    return n * rank // world, n * (rank + 1) // world


def shard_batch(items, world: int, rank: int):
    lo, hi = shard_range(len(items), world, rank)
    return items[lo:hi]


class TorchDistComm:
    """Sum-allreduce through torch.distributed on the current stream."""

    def __init__(self, group=None):
        self.group = group

    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM, group=self.group)
        return t


class LocalComm:
    """World of one: identity."""

    def allreduce(self, t):
        return t


class DeviceShardOps:
    """Per-shard arithmetic on the device through the C ABI (tp_als_shard_*)."""

    def __init__(self, V: CPTensor, r: int):
        self.V, self.r = V, r
        self.L = _lib.lib()
        self.qs = _lib.int_array(V.qs)
        self.d, self.Rl = V.ndim, V.rank
        dev = V.data.device
        self.C = torch.empty((self.d, r, self.Rl), dtype=torch.float64, device=dev)
        self.G = torch.empty((self.d, r, r), dtype=torch.float64, device=dev)
        self.info = torch.zeros(2, dtype=torch.int32, device=dev)
        n = self.L.tp_als_shard_ws_bytes(self.d, self.qs, self.Rl, r)
        if n == 0:
            raise ValueError(f"unsupported shard size d={self.d}, R_l={self.Rl}, r={r} (r <= 32)")
        self.ws = torch.empty(n, dtype=torch.uint8, device=dev)
        self.st = _lib.stream_ptr(dev)

    def init(self, U: torch.Tensor):
        _lib.check(self.L.tp_als_shard_init_f64(self.d, self.qs, self.Rl, self.V.data.data_ptr(), self.r,
                                                U.data_ptr(), self.C.data_ptr(), self.G.data_ptr(), self.st),
                   "shard init")

    def rhs(self, j: int) -> torch.Tensor:
        if not hasattr(self, "_rhs"):
            dev = self.V.data.device
            self._rhs = [torch.empty((self.r, q), dtype=torch.float64, device=dev) for q in self.V.qs]
        out = self._rhs[j]
        _lib.check(self.L.tp_als_shard_rhs_f64(self.d, self.qs, self.Rl, self.V.data.data_ptr(), self.r,
                                               self.C.data_ptr(), j, out.data_ptr(), self.ws.data_ptr(),
                                               self.ws.numel(), self.st), "shard rhs")
        return out

    def update(self, U: torch.Tensor, j: int, rhs: torch.Tensor, reg: float, reg_mode: int):
        _lib.check(self.L.tp_als_shard_update_f64(self.d, self.qs, self.Rl, self.V.data.data_ptr(), self.r,
                                                  U.data_ptr(), self.C.data_ptr(), self.G.data_ptr(), j,
                                                  rhs.data_ptr(), float(reg), int(reg_mode), self.info.data_ptr(),
                                                  self.ws.data_ptr(), self.ws.numel(), self.st), "shard update")

    def check(self):
        if int(self.info[0].item()):
            from .cp import ConditioningError
            raise ConditioningError("regularised normal equations are not positive definite")


class ShardedALS:
    """Fixed-sweep Gauss-Seidel ALS over an R-sharded target (cp.py:310-320 per mode)."""

    def __init__(self, ops, comm=None, config: ALSApproxConfig | None = None):
        self.ops = ops
        self.comm = comm or LocalComm()
        self.cfg = config or ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
        if self.cfg.tol > 0 or self.cfg.stall > -np.inf:
            raise ValueError("the sharded ALS runs a fixed sweep count (tol=0, stall=-inf)")

    def begin(self, U):
        self.U = U
        self.ops.init(U)

    def mode_rhs(self, j):
        return self.ops.rhs(j)

    def mode_finish(self, j, rhs_total):
        reg, mode = (1e-12, 1) if self.cfg.reg is None else (float(self.cfg.reg), 0)
        self.ops.update(self.U, j, rhs_total, reg, mode)

    def run(self, U, d: int):
        """U: replicated guess (modified in place)."""
        self.begin(U)
        for _ in range(self.cfg.max_sweeps):
            for j in range(d):
                rhs = self.mode_rhs(j)
                self.comm.allreduce(rhs)
                self.mode_finish(j, rhs)
        return U

    def capture(self, U, d: int):
        """Record one whole truncation (init + every mode step + all-reduce) into a
        CUDA graph on a side stream; ``replay()`` then runs it with one launch.
        U must keep its address (copy the next initial guess into it)."""
        self.run(U, d)   # warm-up: lazily allocated buffers, NCCL communicator
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            self.ops.st = _lib.stream_ptr(U.device)
            with torch.cuda.graph(self.graph, stream=st):
                self.ops.st = st.cuda_stream
                self.run(U, d)
        torch.cuda.current_stream().wait_stream(st)
        self.ops.st = _lib.stream_ptr(U.device)
        return self.graph

    def replay(self):
        self.graph.replay()


class GraphShardedALS:
    """R-sharded truncation driver: the per-mode-update kernels plus the all-reduce of
    ShardedALS, captured once as a CUDA graph and replayed per truncation."""

    def __init__(self, V_local: CPTensor, r: int, config: ALSApproxConfig | None = None, group=None):
        dist = torch.distributed.is_available() and torch.distributed.is_initialized()
        self.world = torch.distributed.get_world_size(group) if dist else 1
        self.comm = TorchDistComm(group) if dist else LocalComm()
        self.ops = DeviceShardOps(V_local, r)
        self.drv = ShardedALS(self.ops, self.comm, config)
        self.d = V_local.ndim

    def prepare(self, U: torch.Tensor):
        self.U = U
        self.drv.capture(U, self.d)

    def run(self, U: torch.Tensor):
        if U.data_ptr() != self.U.data_ptr():
            raise ValueError("run() needs the buffer prepare() captured")
        self.drv.replay()

    def check(self):
        self.ops.check()

    def describe(self) -> str:
        return "per mode update: shard rhs kernel, NCCL all-reduce of the r x Q block, replicated update; " \
               "one CUDA graph per truncation"

    def kernel_name(self) -> str:
        return "tp_als_shard_* mode steps + NCCL all-reduce (per GPU)"

    def launches_per_truncation(self) -> int:
        return self.drv.cfg.max_sweeps * self.d * 6 + 2 * self.d


class FusedShardedALS:
    """R-sharded truncation in ONE fused launch per GPU (``tp_als_xg_f64``): every
    rank runs the cluster ALS kernel on its R-slab; the per-mode-update r x Q
    right-hand-side exchange happens inside the kernel through peer-mapped
    exchange buffers (CUDA IPC handles swapped once with all_gather_object) and an
    in-kernel cross-GPU barrier (one system-scope arrival per CTA on every rank's counter) -- no
    host round trip or NCCL call per mode update.
    Every rank ends with the identical (bitwise) fit."""

    def __init__(self, V_local: CPTensor, r: int, config: ALSApproxConfig | None = None, group=None):
        import ctypes
        self.cfg = config or ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
        if self.cfg.tol > 0 or self.cfg.stall > -np.inf:
            raise ValueError("the sharded ALS runs a fixed sweep count (tol=0, stall=-inf)")
        dist = torch.distributed.is_available() and torch.distributed.is_initialized()
        self.world = torch.distributed.get_world_size(group) if dist else 1
        self.rank = torch.distributed.get_rank(group) if dist else 0
        self.V, self.r, self.d = V_local, r, V_local.ndim
        self.L = _lib.lib()
        self.qs = _lib.int_array(V_local.qs)
        L = self.L
        nws = L.tp_als_xg_ws_bytes(self.d, self.qs, V_local.rank, r, self.world, 1)
        npeer = L.tp_als_xg_peer_bytes(self.d, self.qs, V_local.rank, r, self.world, 1)
        if nws == 0 or npeer == 0:
            raise ValueError(f"unsupported sharded ALS size d={self.d}, R_l={V_local.rank}, r={r}")
        dev = V_local.data.device
        self.ws = torch.empty(nws, dtype=torch.uint8, device=dev)
        self.info = torch.zeros(2, dtype=torch.int32, device=dev)
        ptr = ctypes.c_void_p()
        _lib.check(L.tp_dev_alloc(npeer, ctypes.byref(ptr)), "exchange buffer")
        self._mine = ptr.value
        self._opened = []
        peers = [self._mine]
        if self.world > 1:
            h = (ctypes.c_char * 64)()
            _lib.check(L.tp_ipc_handle(self._mine, h), "ipc handle")
            handles = [None] * self.world
            torch.distributed.all_gather_object(handles, bytes(h), group=group)
            peers = []
            for i, hb in enumerate(handles):
                if i == self.rank:
                    peers.append(self._mine)
                    continue
                p2 = ctypes.c_void_p()
                _lib.check(L.tp_ipc_open(ctypes.c_char_p(hb), ctypes.byref(p2)), "ipc open")
                self._opened.append(p2.value)
                peers.append(p2.value)
        self._peers = (ctypes.c_void_p * self.world)(*peers)
        self.group = group
        plan = (ctypes.c_int * 4)()
        _lib.check(L.tp_als_xg_plan(self.d, self.qs, V_local.rank, r, self.world, 1, plan), "plan")
        self.plan = {"ctas": plan[0], "cluster": plan[1], "clusters": plan[2], "smem_bytes": plan[3]}

    def prepare(self, U: torch.Tensor):
        pass

    def run(self, U: torch.Tensor, V: CPTensor | None = None):
        import ctypes
        V = V or self.V
        if V.rank != self.V.rank or V.qs != self.V.qs:
            raise ValueError("slab shape differs from the planned one")
        reg, mode = (1e-12, 1) if self.cfg.reg is None else (float(self.cfg.reg), 0)
        one = lambda v: (ctypes.c_void_p * 1)(v)   # noqa: E731
        st = self.L.tp_als_xg_f64(self.d, self.qs, V.rank, self.r, int(self.cfg.max_sweeps), reg, mode, 1,
                                  one(V.data.data_ptr()), one(U.data_ptr()), one(self.info.data_ptr()),
                                  one(self.ws.data_ptr()), self.ws.numel(), self.world, self.rank, self._peers,
                                  _lib.stream_ptr(U.device))
        _lib.check(st, "sharded cp_approx_als")
        return U

    def check(self):
        _check_xg_info(self.info)

    def describe(self) -> str:
        return (f"one fused launch per GPU: {self.plan['clusters']} clusters x {self.plan['cluster']} CTAs on the "
                f"rank's R-slab, in-kernel exchange of the r x Q partials through peer-mapped memory, cross-GPU "
                f"counter barrier once per mode update")

    def kernel_name(self) -> str:
        return f"tp::als_xg<32> ({self.plan['ctas']} CTAs per GPU, cluster {self.plan['cluster']})"

    def launches_per_truncation(self) -> int:
        return 1

    def close(self):
        if self._mine is None:
            return
        torch.cuda.synchronize()
        if self.world > 1:
            torch.distributed.barrier(group=self.group)
        for p in self._opened:
            self.L.tp_ipc_close(p)
        self._opened = []
        self.L.tp_dev_free(self._mine)
        self._mine = None

    def __del__(self):
        try:
            if self._mine is not None and self.world == 1:
                self.L.tp_dev_free(self._mine)
                self._mine = None
        except Exception:
            pass


def _check_xg_info(info: torch.Tensor) -> None:
    from .cp import ConditioningError
    status = int(info[0].item())
    if status & 4:
        raise RuntimeError("sharded ALS: a peer rank did not reach the exchange barrier within 5 s")
    if status & 2:
        raise ConditioningError("normal equations produced non-finite coefficients")
    if status & 1:
        raise ConditioningError("regularised normal equations are not positive definite")


def make_sharded_als(V_local: CPTensor, r: int, config: ALSApproxConfig | None = None, group=None,
                     impl: str = "auto"):
    """The R-sharded truncation driver: the fused one-launch kernel (``impl="fused"``,
    the default when the size is supported) or the per-mode kernels + NCCL graph."""
    if impl in ("auto", "fused"):
        try:
            return FusedShardedALS(V_local, r, config, group)
        except ValueError:
            if impl == "fused":
                raise
    return GraphShardedALS(V_local, r, config, group)


_DRIVERS: dict = {}


def sharded_cp_approx_als(V_local: CPTensor, init: CPTensor, config: ALSApproxConfig | None = None,
                          group=None, check: bool = True) -> CPTensor:
    """R-sharded ``cp_approx_als``: every rank passes its slab of the target and the
    same initial guess; every rank gets the full fit.  The fused driver (and its
    peer mappings) is cached per (shapes, config, group); ``check=False`` defers
    the status read (no host round trip)."""
    cfg = config or ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
    key = (V_local.qs, V_local.rank, init.rank, cfg.max_sweeps, cfg.reg, id(group), V_local.data.device.index)
    drv = _DRIVERS.get(key)
    if drv is None:
        try:
            drv = FusedShardedALS(V_local, init.rank, cfg, group)
        except ValueError:
            drv = None
        _DRIVERS[key] = drv
    out = init.copy()
    if drv is None:
        comm = TorchDistComm(group) if (torch.distributed.is_available() and torch.distributed.is_initialized()) \
            else LocalComm()
        ops = DeviceShardOps(V_local, init.rank)
        ShardedALS(ops, comm, cfg).run(out.data, init.ndim)
        if check:
            ops.check()
        return out
    drv.run(out.data, V_local)
    if check:
        drv.check()
    return out


def simulate_sharded_als(V_factors, init_factors, shards: int, config: ALSApproxConfig | None = None,
                         specs=None):
    """Run the fused R-sharded kernel with ``shards`` ranks' CTA groups co-resident in
    ONE launch on this GPU (each group its own slab, replicated state and exchange
    buffer; the in-kernel exchange and barrier work exactly as across GPUs).
    Returns the per-rank fits (device tensors in CP layout)."""
    import ctypes
    from .basis import BasisSpec
    cfg = config or ALSApproxConfig(max_sweeps=20, stall=-np.inf, reg=1e-10)
    V_factors = [np.asarray(v) for v in V_factors]
    qs = [v.shape[0] for v in V_factors]
    R = V_factors[0].shape[1]
    r = init_factors[0].shape[1]
    specs = specs or tuple(BasisSpec(q, np.pi, "collocation", lo=0.0) for q in qs)
    L = _lib.lib()
    d = len(qs)
    spans = [shard_range(R, shards, g) for g in range(shards)]
    if len({hi - lo for lo, hi in spans}) != 1:
        raise ValueError("simulated shards need equal slabs (R divisible by shards)")
    Rl = spans[0][1] - spans[0][0]
    qa = _lib.int_array(qs)
    nws = L.tp_als_xg_ws_bytes(d, qa, Rl, r, shards, shards)
    npeer = L.tp_als_xg_peer_bytes(d, qa, Rl, r, shards, shards)
    if nws == 0 or npeer == 0:
        raise ValueError("unsupported simulated sharded ALS size")
    dev = _lib.device()
    Vs = [CPTensor(specs, [v[:, lo:hi] for v in V_factors]) for lo, hi in spans]
    Us = [CPTensor(specs, init_factors).data for _ in range(shards)]
    infos = [torch.zeros(2, dtype=torch.int32, device=dev) for _ in range(shards)]
    wss = [torch.empty(nws, dtype=torch.uint8, device=dev) for _ in range(shards)]
    peers = [torch.zeros(npeer, dtype=torch.uint8, device=dev) for _ in range(shards)]
    arr = lambda ts: (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])   # noqa: E731
    reg, mode = (1e-12, 1) if cfg.reg is None else (float(cfg.reg), 0)
    st = L.tp_als_xg_f64(d, qa, Rl, r, int(cfg.max_sweeps), reg, mode, shards, arr([v.data for v in Vs]), arr(Us),
                         arr(infos), arr(wss), nws, shards, 0, arr(peers), _lib.stream_ptr(dev))
    _lib.check(st, "simulated sharded ALS")
    for inf in infos:
        _check_xg_info(inf)
    return Us
