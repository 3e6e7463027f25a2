"""cfg4 hSVD batch time per batched-GEMM kernel variant (debug hook)."""
import ctypes, runpy, sys
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402
L = _lib.lib()
L.tp_debug_set_bgemm_variant.argtypes = [ctypes.c_int]
for v in [int(x) for x in sys.argv[1:]] or [0, 1, 2, 3, 4]:
    L.tp_debug_set_bgemm_variant(v)
    sys.argv = ["ht_timing.py", "64"]
    print(f"bgemm variant {v}: ", end="", flush=True)
    runpy.run_path("tools/ht_timing.py", run_name="__main__")
L.tp_debug_set_bgemm_variant(1)
