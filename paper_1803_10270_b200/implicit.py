"""Fixed-rank implicit time stepping by (damped) alternating least squares
(mirror of ``tensorpde/implicit.py``).

``step`` runs every sweep of one implicit step in ``tp_implicit_step_f64``:
device assembly of the normal-equation blocks M_q / gamma_q (implicit.py:125-153),
a hand-written blocked Cholesky solve of (M_q + lam I) x = gamma_q (replacing the
LSQR of implicit.py:156-164; SURVEY 8(c) shim S6), the convergence measure and
damping (implicit.py:167-177, 281-282).  ``orientation="corrected"`` assembles
the true normal equations of min |A f_new - B f_old|^2; ``"reference"``
reproduces build_gamma's pairing (implicit.py:137-139).
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import StepFailure
from .basis import BasisSpec
from .cp import CPTensor
from .operators import CrankNicolsonPair, dense_factor

__all__ = ["ALSStepConfig", "OperatorTables", "StepWorkspace", "StepFailure", "build_tables", "step"]

logger = logging.getLogger(__name__)


@dataclass
class ALSStepConfig:
    """implicit.py:59-74, plus ``lam`` (Tikhonov constant of the direct solve) and
    ``orientation`` ("corrected" | "reference")."""

    dt: float
    eps_tol: float = 1e-8
    max_sweeps: int = 500
    delta_beta: float = 4.0
    lsqr_tol: float = 1e-12
    lsqr_maxit: int = 2000
    workers: int = 1
    schedule: str = "jacobi"
    lam: float = 1e-10
    orientation: str = "corrected"
    solver: str = "auto"        # "auto" | "dense" | "circulant"

    def __post_init__(self):
        if self.schedule not in ("jacobi", "gauss-seidel"):
            raise ValueError(f"unknown schedule {self.schedule!r}")
        if self.delta_beta < 1.0:
            raise ValueError("damping divisor must be >= 1")
        if self.orientation not in ("corrected", "reference"):
            raise ValueError(f"unknown orientation {self.orientation!r}")
        if self.solver not in ("auto", "dense", "circulant"):
            raise ValueError(f"unknown solver {self.solver!r}")


@dataclass
class OperatorTables:
    """Deduplicated pairing tables pairs[k][e][z] = F_{e,k}^T F_{z,k} (implicit.py:77-108)."""

    pair: CrankNicolsonPair
    tabs: torch.Tensor          # (n_tab, Q, Q) device
    tab_id: np.ndarray          # (d, ra, ra) int32
    KL: np.ndarray
    KR: np.ndarray
    circ_eig: torch.Tensor | None = None   # (n_tab, Q, 2) eigenvalues if every table is circulant
    qs: tuple = ()                          # true mode sizes (modes zero-padded to max(qs) when they differ)

    def _replace_qs(self) -> "OperatorTables":
        """The same tables for the padded (uniform) launch."""
        from dataclasses import replace
        return replace(self, qs=())


def build_tables(pair: CrankNicolsonPair, device=None) -> OperatorTables:
    """Pairing tables pairs[k][e][z] = E_{e,k}^T E_{z,k} (implicit.py:77-108), deduplicated.
    Modes of different sizes are zero-padded to Q = max Q_k: a padded table is zero on the
    padding rows/columns, so the padded normal equations decouple there (lambda I, zero
    right-hand side) and the padding rows of the iterate stay exactly zero."""
    specs = pair.specs
    qtrue = tuple(s.Q for s in specs)
    Q = max(qtrue)
    if any(s.kind == "fourier" for s in specs):
        # the reference's Galerkin pair_matrix is the unconjugated bilinear form of a complex
        # basis (basis.py:207-214; the identity pairs to the flip matrix), not E_e^T E_z
        raise ValueError("the B200 implicit step runs on real collocation/uniform grids; "
                         "Fourier Galerkin specs (complex pairing tables) are not supported")
    ra, d = pair.n_terms, len(specs)
    uniq, keys, tab_id = [], {}, np.zeros((d, ra, ra), dtype=np.int32)
    for k, spec in enumerate(specs):
        mats = []
        for e in range(ra):
            m = dense_factor(spec, pair.factors[e][k])
            if m is not None and np.iscomplexobj(m):
                raise ValueError("complex factor matrices are not supported by the real-fp64 implicit step")
            mats.append(np.eye(spec.Q) if m is None else m)
        for e in range(ra):
            for z in range(ra):
                t = np.zeros((Q, Q))
                t[:spec.Q, :spec.Q] = mats[e].T @ mats[z]
                key = t.tobytes()
                if key not in keys:
                    keys[key] = len(uniq)
                    uniq.append(t)
                tab_id[k, e, z] = keys[key]
    eta = np.asarray([complex(x) for x in pair.eta])
    zeta = np.asarray([complex(x) for x in pair.zeta])
    if np.any(eta.imag != 0) or np.any(zeta.imag != 0):
        raise ValueError("complex operator weights are not supported on the real-fp64 B200 path")
    eta, zeta = eta.real, zeta.real
    dev = device or _lib.device()
    tabs = torch.as_tensor(np.stack(uniq)).to(dev)
    circ = None
    if all(is_circulant(t) for t in uniq):
        lam = np.stack([np.fft.fft(t[:, 0]) for t in uniq])          # lambda_t(k) = sum_m t[m,0] e^{-2 pi i mk/Q}
        circ = torch.as_tensor(np.stack([lam.real, lam.imag], axis=-1)).to(dev)
    return OperatorTables(pair, tabs, tab_id, np.outer(eta, eta), np.outer(eta, zeta), circ, qtrue)


def is_circulant(t: np.ndarray, rtol: float = 1e-13) -> bool:
    """t[i][j] depends only on (i - j) mod Q (periodic collocation operators)."""
    Q = t.shape[0]
    col = t[:, 0]
    idx = (np.arange(Q)[:, None] - np.arange(Q)[None, :]) % Q
    return bool(np.max(np.abs(t - col[idx])) <= rtol * max(np.max(np.abs(t)), 1e-300))


class StepWorkspace:
    """implicit.py:180-210: reusable tables for repeated steps with one pair."""

    def __init__(self, pair: CrankNicolsonPair, config: ALSStepConfig):
        if abs(config.dt - pair.dt) > 1e-15 * max(abs(pair.dt), 1.0):
            raise ValueError(f"config dt {config.dt} != operator pair dt {pair.dt}")
        self.pair = pair
        self.config = config
        self.tables = build_tables(pair)

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


def _check_forcing(forcing: CPTensor | None, f_n: CPTensor, pair: CrankNicolsonPair) -> None:
    if forcing is None:
        return
    if not isinstance(forcing, CPTensor):
        raise TypeError("forcing must be a CPTensor")
    if forcing.specs != f_n.specs:
        raise ValueError("forcing lives on a different basis")
    if forcing.is_complex:
        raise ValueError("complex128 forcing is not supported by the real-fp64 implicit step")
    if any(dense_factor(s, m) is not None for s, m in zip(pair.specs, pair.factors[0])):
        # the source tables pair(E_e, I) are read as pairs[k][e][0]
        raise ValueError("forcing needs term 0 of the pair to be the identity (crank_nicolson_pair layout)")


def _launch(f_n: CPTensor, out: torch.Tensor, tab: OperatorTables, cfg: ALSStepConfig, eps: torch.Tensor,
            info: torch.Tensor, forcing: CPTensor | None = None) -> None:
    if f_n.is_complex:
        raise ValueError("complex128 states are not supported by the real-fp64 implicit step")
    L = _lib.lib()
    d, r, ra = f_n.ndim, f_n.rank, tab.pair.n_terms
    Q = max(tab.qs) if tab.qs else f_n.specs[0].Q
    if tab.qs and len(set(tab.qs)) > 1:   # zero-padded modes (build_tables): pad in, solve, unpad
        fp = _pad_modes(f_n, Q)
        outp = fp.data.clone()
        fcp = _pad_modes(forcing, Q) if forcing is not None else None
        _launch(fp, outp.view(-1), tab._replace_qs(), cfg, eps, info, fcp)
        _unpad_modes(outp, f_n, Q, out)
        return
    n_tab = tab.tabs.shape[0]
    rf = forcing.rank if forcing is not None else 0
    use_circ = tab.circ_eig is not None and cfg.solver in ("auto", "circulant")
    if cfg.solver == "circulant" and tab.circ_eig is None:
        raise ValueError("solver='circulant' needs circulant pairing tables (periodic collocation factors)")
    nbytes = L.tp_implicit_ws_bytes(d, Q, r, n_tab, ra, rf)
    if nbytes == 0:
        raise ValueError(f"unsupported implicit-step size d={d}, Q={Q}, r={r}, tables={n_tab}")
    ws = _lib.WORKSPACE.get(nbytes, f_n.data.device)
    st = L.tp_implicit_step_f64(d, Q, r, ra, n_tab, tab.tabs.data_ptr(), _lib.int_array(tab.tab_id.reshape(-1)),
                                _lib.double_array(tab.KL.reshape(-1)), _lib.double_array(tab.KR.reshape(-1)),
                                f_n.data.data_ptr(), out.data_ptr(), int(cfg.max_sweeps),
                                0 if cfg.schedule == "gauss-seidel" else 1, float(cfg.delta_beta),
                                float(cfg.eps_tol), float(cfg.lam), 1 if cfg.orientation == "reference" else 0,
                                tab.circ_eig.data_ptr() if use_circ else None,
                                forcing.data.data_ptr() if rf else None, rf,
                                _lib.double_array([tab.pair.dt * float(complex(x).real) for x in tab.pair.eta]),
                                eps.data_ptr(), info.data_ptr(), ws.data_ptr(), ws.numel(),
                                _lib.stream_ptr(f_n.data.device))
    _lib.check(st, "implicit.step")


def _pad_modes(f: CPTensor, Q: int) -> CPTensor:
    """Mode-major copy with every mode zero-padded to Q rows (device copies)."""
    r = f.rank
    out = torch.zeros(len(f.specs) * Q * r, dtype=f.data.dtype, device=f.data.device)
    off = 0
    for k, s in enumerate(f.specs):
        out[k * Q * r:k * Q * r + s.Q * r] = f.data[off:off + s.Q * r]
        off += s.Q * r
    return CPTensor(tuple(BasisSpec(Q, 1.0, "collocation") for _ in f.specs), data=out, rank=r)


def _unpad_modes(src: torch.Tensor, like: CPTensor, Q: int, out: torch.Tensor) -> None:
    r, off = like.rank, 0
    for k, s in enumerate(like.specs):
        out[off:off + s.Q * r] = src[k * Q * r:k * Q * r + s.Q * r]
        off += s.Q * r


def step(f_n: CPTensor, pair: CrankNicolsonPair, forcing: CPTensor | None, config: ALSStepConfig,
         workspace: StepWorkspace | None = None, log: dict | None = None) -> CPTensor:
    """Advance one implicit step at fixed separation rank (implicit.py:222-301), with the
    source term ``forcing`` (implicit.py:140-152) when given.

    ``log`` receives the reference's keys (implicit.py:289-297): ``sweeps``,
    ``eps_conv`` and ``converged`` as computed on the device, ``solve_seconds`` =
    device time of the whole step (CUDA events; assembly and solve are fused
    into the same kernels, so ``assembly_seconds`` is None), ``lsqr_iterations``
    None (direct Cholesky solves) and ``direct_solves`` = sweeps x d."""
    ws = workspace or StepWorkspace(pair, config)
    _check_forcing(forcing, f_n, pair)
    dev = f_n.data.device
    out = f_n.data.clone()
    eps = torch.full((1,), float("inf"), dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _launch(f_n, out, ws.tables, config, eps, info, forcing)
    e1.record()
    status, sweeps = (int(v) for v in info.tolist())
    eps_conv = float(eps.item())
    if status & 2:
        raise StepFailure(-1, sweeps, float("nan"))
    if status & 1:
        raise StepFailure(-1, sweeps, float("inf"))
    did_converge = eps_conv <= config.eps_tol
    if not did_converge:
        logger.warning("sweep cap %d hit with update %.3e > %.3e", config.max_sweeps, eps_conv, config.eps_tol)
    if log is not None:
        e1.synchronize()
        log.update(sweeps=sweeps, eps_conv=eps_conv, converged=did_converge, assembly_seconds=None,
                   solve_seconds=e0.elapsed_time(e1) / 1e3, lsqr_iterations=None, direct_solves=sweeps * f_n.ndim)
    return CPTensor(f_n.specs, data=out, rank=f_n.rank)


def run(f0: CPTensor, pair: CrankNicolsonPair, config: ALSStepConfig, steps: int,
        workspace: StepWorkspace | None = None, forcing: CPTensor | None = None) -> CPTensor:
    """``steps`` implicit steps, stream-ordered (no host synchronisation inside a step;
    convergence is decided on the device), one status check at the end."""
    ws = workspace or StepWorkspace(pair, config)
    _check_forcing(forcing, f0, pair)
    dev = f0.data.device
    eps = torch.zeros(1, dtype=torch.float64, device=dev)
    infos = torch.zeros((max(steps, 1), 2), dtype=torch.int32, device=dev)
    cur = f0
    for n in range(steps):
        out = cur.data.clone()
        _launch(cur, out, ws.tables, config, eps, infos[n], forcing)
        cur = CPTensor(f0.specs, data=out, rank=f0.rank)
    bad = int(infos[:, 0].max().item())
    if bad:
        raise StepFailure(-1, config.max_sweeps, float("nan"))
    return cur
