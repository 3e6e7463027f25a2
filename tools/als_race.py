"""Race detector: the fused ALS kernels are deterministic for a fixed plan, so repeated
runs must be bitwise identical.  python tools/als_race.py [reps] [var:grid ...]"""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1803_10270_b200 import _lib, cp  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402

L = _lib.lib()
L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
combos = [tuple(int(v) for v in c.split(":")) for c in sys.argv[2:]] or [(0, 0)]
g = np.load("tests/golden/cp_als.npz")
cases = []
n = "r32_q64"
cases.append(([g[f"{n}_V_{k}"] for k in range(4)], [g[f"{n}_init_{k}"] for k in range(4)], 6, 32))
rng = np.random.default_rng(0)
V = [rng.standard_normal((64, 588)) / 8 for _ in range(6)]
cases.append((V, [v[:, :12].copy() for v in V], 10, 12))
V = [rng.standard_normal((256, 512)) / 16 for _ in range(6)]
cases.append((V, [v[:, :32].copy() for v in V], 20, 32))
for var, grid in combos:
    L.tp_debug_set_als_variant(var if var != 2 else 2, grid if var == 2 else 0)
    for ci, (V, I, sweeps, r) in enumerate(cases):
        S = tuple(BasisSpec(v.shape[0], np.pi, "collocation", lo=0.0) for v in V)
        T, I0 = cp.CPTensor(S, V), cp.CPTensor(S, I)
        cfg = cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10, grid=0 if var == 2 else grid)
        for tr in (None, []):
            try:
                first = cp.cp_approx_als(T, r, cfg, init=I0, trace=tr).data.clone()
            except Exception as e:  # noqa: BLE001
                print(var, grid, ci, "skip:", e); break
            bad, worst = 0, 0.0
            for _ in range(reps):
                out = cp.cp_approx_als(T, r, cfg, init=I0, trace=tr).data
                if not torch.equal(out, first):
                    bad += 1
                    worst = max(worst, float((out - first).abs().max() / first.abs().max()))
            print(f"var {var} grid {grid} case {ci} trace {tr is not None}: {bad}/{reps} differ (worst {worst:.2e})", flush=True)
L.tp_debug_set_als_variant(0, 0)
