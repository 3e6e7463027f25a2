"""cfg4 hSVD time and Jacobi sweep counts vs rotation threshold (debug hook)."""
import ctypes
import subprocess
import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402
L = _lib.lib()
L.tp_debug_set_jacobi.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
for tol in [1e-16, 2.3e-16, 1e-15, 1e-14]:
    L.tp_debug_set_jacobi(30, tol, cnt.data_ptr())
    cnt.zero_()
    import runpy
    sys.argv = ["ht_timing.py", "64"]
    runpy.run_path("tools/ht_timing.py", run_name="__main__")
    torch.cuda.synchronize()
    print(f"  tol {tol:.1e}: avg sweeps per matrix {cnt.item() / (8 * 2 * 896):.2f}", flush=True)
