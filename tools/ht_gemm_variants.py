"""Config-4 batch time per batched-GEMM kernel variant (tp_debug_set_bgemm_variant)."""
import ctypes
import subprocess
import sys
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402
L = _lib.lib()
L.tp_debug_set_bgemm_variant.argtypes = [ctypes.c_int]
import runpy  # noqa: E402
for v in (1, 2, 3, 4):
    L.tp_debug_set_bgemm_variant(v)
    print("variant", v, end=": ", flush=True)
    runpy.run_path("tools/ht_timing.py", run_name="__main__")
L.tp_debug_set_bgemm_variant(1)
