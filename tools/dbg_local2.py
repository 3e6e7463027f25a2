import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import cp_als as ocp, metrics
from paper_1803_10270_b200 import cp
from paper_1803_10270_b200.basis import BasisSpec
for qs, R, r in [((5, 5, 5), 6, 2), ((5, 7, 3), 6, 2), ((7, 7, 7), 6, 2), ((5, 7, 3), 6, 4), ((8, 8, 8), 6, 2), ((9, 9, 9), 6, 2), ((12, 12, 12), 6, 2), ((16, 16, 16), 6, 2)]:
    rng = np.random.default_rng(1)
    V = [rng.standard_normal((q, R)) for q in qs]
    init = [v[:, :r].copy() for v in V]
    S = tuple(BasisSpec(q, np.pi, "collocation", lo=0.0) for q in qs)
    for grid in (0, 2):
        cfg = cp.ALSApproxConfig(max_sweeps=5, tol=0.0, stall=-np.inf, reg=1e-10, grid=grid)
        out = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init))
        ref = ocp.als(V, init, 5, lam=1e-10)
        print(qs, R, r, "grid", grid, cp.als_plan(list(qs), R, r, grid)["ctas"], metrics.cp_rel_diff(ref, out.to_numpy()))
