"""cfg4 hSVD batch time with each Jacobi kernel (debug hook tp_debug_set_jacobi_impl)."""
import ctypes
import runpy
import sys
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402
L = _lib.lib()
L.tp_debug_set_jacobi_impl.argtypes = [ctypes.c_int]
L.tp_debug_set_jacobi.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p]
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
for impl in [0, 2, 0, 2]:
    L.tp_debug_set_jacobi_impl(impl)
    L.tp_debug_set_jacobi(30, 1e-16, cnt.data_ptr())
    cnt.zero_()
    sys.argv = ["ht_timing.py", "64"]
    print(f"impl {impl}: ", end="", flush=True)
    runpy.run_path("tools/ht_timing.py", run_name="__main__")
    torch.cuda.synchronize()
    print(f"   avg sweeps per matrix {cnt.item() / (8 * 896):.2f}", flush=True)
