"""cfg4 batch time with / without the K-contiguous shared layout (debug hook)."""
import ctypes, runpy, sys
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402
L = _lib.lib()
L.tp_debug_set_bgemm_klayout.argtypes = [ctypes.c_int]
for on in (0, 1, 0, 1):
    L.tp_debug_set_bgemm_klayout(on)
    sys.argv = ["ht_timing.py", "64"]
    print(f"klayout {on}: ", end="", flush=True)
    runpy.run_path("tools/ht_timing.py", run_name="__main__")
L.tp_debug_set_bgemm_klayout(1)
