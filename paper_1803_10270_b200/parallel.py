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

__all__ = ["shard_range", "ShardedALS", "DeviceShardOps", "TorchDistComm", "LocalComm", "shard_batch"]


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


def make_sharded_als(V_local: CPTensor, r: int, config: ALSApproxConfig | None = None, group=None):
    """The R-sharded truncation driver for this process group."""
    return GraphShardedALS(V_local, r, config, group)


def sharded_cp_approx_als(V_local: CPTensor, init: CPTensor, config: ALSApproxConfig | None = None,
                          group=None, check: bool = True) -> CPTensor:
    """R-sharded ``cp_approx_als``: every rank passes its slab of the target and the
    same initial guess; every rank gets the full fit.  ``check=False`` defers the
    status read (no host round trip)."""
    comm = TorchDistComm(group) if (torch.distributed.is_available() and torch.distributed.is_initialized()) \
        else LocalComm()
    ops = DeviceShardOps(V_local, init.rank)
    out = init.copy()
    ShardedALS(ops, comm, config).run(out.data, init.ndim)
    if check:
        ops.check()
    return out
