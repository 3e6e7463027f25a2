"""A/B the node-Gram eigensolver at config 4 (tridiagonal vs Jacobi): batch time."""
import ctypes
import subprocess
import sys
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib  # noqa: E402

L = _lib.lib()
L.tp_debug_set_eig_tridiag.argtypes = [ctypes.c_int]
for on in (1, 0, 1):
    L.tp_debug_set_eig_tridiag(on)
    print("tridiag" if on else "jacobi ", end=": ", flush=True)
    exec(open("tools/ht_timing.py").read())
