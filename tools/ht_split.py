"""cfg4 batch time vs the split-K wave target (debug hook)."""
import ctypes, runpy, sys
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402
L = _lib.lib()
L.tp_debug_set_ht_split_waves.argtypes = [ctypes.c_int]
for w in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
    L.tp_debug_set_ht_split_waves(w)
    sys.argv = ["ht_timing.py", "64"]
    print(f"split waves {w}: ", end="", flush=True)
    runpy.run_path("tools/ht_timing.py", run_name="__main__")
L.tp_debug_set_ht_split_waves(4)
