"""ctypes binding of the sm_100a C-ABI library (include/tpde_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises.  Status codes map onto the reference's exceptions
(SURVEY.md 8(b)): TP_EINVAL/TP_EUNSUPPORTED -> ValueError, TP_ENONFINITE /
TP_ENOTPD -> ConditioningError (cp.py:38-39, 178-179), TP_ECUDA /
TP_EWORKSPACE -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import warnings
import re
from pathlib import Path

import torch

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libtpde_b200.so"
HEADER = PKG.parent / "include" / "tpde_b200.h"

TP_OK, TP_EINVAL, TP_ENONFINITE, TP_ENOTPD, TP_ECUDA, TP_EWORKSPACE, TP_EUNSUPPORTED = range(7)


class ConditioningError(RuntimeError):
    """Normal equations unsalvageably singular or non-finite (cp.py:38-39)."""


class StepFailure(RuntimeError):
    """A per-dimension implicit solve broke down (implicit.py:51-56)."""

    def __init__(self, dim: int, itn: int, residual: float):
        self.dim, self.itn, self.residual = dim, itn, residual
        super().__init__(f"solve failed in dimension {dim}: itn={itn}, residual={residual:.3e}")


_lib = None

_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_ll_p = ctypes.POINTER(ctypes.c_longlong)
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int
_d = ctypes.c_double

_SIGNATURES = {
    "tp_version": (ctypes.c_char_p, []),
    "tp_status_string": (ctypes.c_char_p, [_i]),
    "tp_last_error": (ctypes.c_char_p, []),
    "tp_device_sms": (_i, []),
    "tp_cp_inner_ws_bytes": (_sz, [_i, _c_int_p, _i, _i]),
    "tp_cp_inner_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _i, _vp, _vp, _sz, _vp]),
    "tp_cp_als_ws_bytes": (_sz, [_i, _c_int_p, _i, _i, _i]),
    "tp_cp_als_plan": (_i, [_i, _c_int_p, _i, _i, _i, _c_int_p]),
    "tp_cp_als_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _i, _d, _i, _d, _d, _vp, _vp, _i, _vp, _sz, _vp]),
    "tp_cp_als_recipe_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _d, _vp, _d, _i, _i, _c_double_p, _c_int_p, _vp,
                                  _c_ll_p, _i, _vp, _i, _d, _i, _vp, _vp, _sz, _vp]),
    "tp_cp_contract_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _vp, _vp]),
    "tp_cp_apply_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _c_double_p, _d, _c_int_p, _vp, _c_ll_p, _i,
                             _vp, _i, _i, _vp]),
    "tp_cp_apply_c128": (_i, [_i, _c_int_p, _i, _vp, _i, _c_double_p, _d, _d, _c_int_p, _vp, _c_ll_p, _i,
                              _vp, _i, _i, _vp]),
    "tp_cp_inner_c128_ws_bytes": (_sz, [_i, _c_int_p, _i, _i]),
    "tp_cp_inner_c128": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _vp, _vp, _sz, _vp]),
    "tp_cp_als_c128_ws_bytes": (_sz, [_i, _c_int_p, _i, _i]),
    "tp_cp_als_c128": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _i, _d, _i, _d, _d, _vp, _vp, _vp, _sz, _vp]),
    "tp_als_shard_ws_bytes": (_sz, [_i, _c_int_p, _i, _i]),
    "tp_als_shard_init_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _vp, _vp, _vp]),
    "tp_als_shard_rhs_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _i, _vp, _vp, _sz, _vp]),
    "tp_als_shard_update_f64": (_i, [_i, _c_int_p, _i, _vp, _i, _vp, _vp, _vp, _i, _vp, _d, _i, _vp, _vp, _sz,
                                     _vp]),
    "tp_als_xg_ws_bytes": (_sz, [_i, _c_int_p, _i, _i, _i, _i]),
    "tp_als_xg_peer_bytes": (_sz, [_i, _c_int_p, _i, _i, _i, _i]),
    "tp_als_xg_plan": (_i, [_i, _c_int_p, _i, _i, _i, _i, _c_int_p]),
    "tp_als_xg_f64": (_i, [_i, _c_int_p, _i, _i, _i, _d, _i, _i, _vp, _vp, _vp, _vp, _sz, _i, _i, _vp, _vp]),
    "tp_dev_alloc": (_i, [_sz, _vp]),
    "tp_dev_free": (_i, [_vp]),
    "tp_ipc_handle": (_i, [_vp, _vp]),
    "tp_ipc_open": (_i, [_vp, _vp]),
    "tp_ipc_close": (_i, [_vp]),
    "tp_ht_truncate_ws_bytes": (_sz, [_i, _i, _i, _i]),
    "tp_ht_truncate_tree_ws_bytes": (_sz, [_i, _c_int_p, _c_int_p, _c_int_p, _i, _i, _i]),
    "tp_ht_truncate_tree_f64": (_i, [_i, _c_int_p, _c_int_p, _c_int_p, _i, _i, _i, _vp, _vp, _i, _d, _vp, _vp, _vp,
                                     _vp, _vp, _vp, _sz, _vp]),
    "tp_ht_truncate_f64": (_i, [_i, _i, _i, _i, _vp, _vp, _i, _d, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "tp_implicit_ws_bytes": (_sz, [_i, _i, _i, _i, _i, _i]),
    "tp_implicit_step_f64": (_i, [_i, _i, _i, _i, _i, _vp, _c_int_p, _c_double_p, _c_double_p, _vp, _vp, _i, _i,
                                  _d, _d, _d, _i, _vp, _vp, _i, _c_double_p, _vp, _vp, _vp, _sz, _vp]),
}


def header_symbols() -> list[str]:
    """Function names declared in include/tpde_b200.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", text)))


def lib():
    """Load (building first if needed) the C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() or os.environ.get("TPDE_REBUILD"):
        from . import build
        build.build()
    if not LIB_PATH.exists():
        raise RuntimeError(f"tpde_b200 CUDA library missing at {LIB_PATH}; run __graft_entry__.build()")
    from . import build
    if build.needs_build():
        # not rebuilt implicitly (a copied tree can carry arbitrary mtimes); say so loudly
        warnings.warn(f"{LIB_PATH.name} is older than its CUDA sources; run __graft_entry__.build() "
                      "or set TPDE_REBUILD=1", RuntimeWarning, stacklevel=2)
    handle = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return handle


def device() -> torch.device:
    """The CUDA device the product path runs on (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1803_10270_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(dev=None) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def check(status: int, what: str = "") -> None:
    if status == TP_OK:
        return
    msg = lib().tp_status_string(status).decode()
    if status == TP_ECUDA:
        msg += ": " + lib().tp_last_error().decode()
    msg = f"{what}: {msg}" if what else msg
    if status in (TP_EINVAL, TP_EUNSUPPORTED):
        raise ValueError(msg)
    if status in (TP_ENONFINITE, TP_ENOTPD):
        raise ConditioningError(msg)
    raise RuntimeError(msg)


def int_array(vals):
    arr = (ctypes.c_int * len(vals))(*[int(v) for v in vals])
    return arr


def double_array(vals):
    return (ctypes.c_double * len(vals))(*[float(v) for v in vals])


def ll_array(vals):
    return (ctypes.c_longlong * len(vals))(*[int(v) for v in vals])


class Workspace:
    """Grow-only per-device scratch buffer (caller-provided workspace of the C ABI)."""

    def __init__(self):
        self._buf = {}

    def get(self, nbytes: int, dev: torch.device) -> torch.Tensor:
        key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            self._buf[key] = buf
        return buf


WORKSPACE = Workspace()
