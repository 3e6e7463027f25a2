"""Debug: hSVD with k > Q leaves (tests/test_gpu_ht.py::test_node_gram_eigensolvers[3-30-33-33])."""
import math
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import ht_hsvd as oht, metrics
from paper_1803_10270_b200 import ht
from paper_1803_10270_b200.basis import BasisSpec

for (d, q, k, rmax) in [(3, 30, 33, 33), (3, 30, 33, 30), (3, 30, 33, 20), (3, 30, 30, 30), (4, 9, 12, 12)]:
    rng = np.random.default_rng(200 + k)
    nodes = oht.balanced_tree(d)
    frames = [None] * len(nodes)
    transfers = [None] * len(nodes)
    for i, nd in enumerate(nodes):
        if oht.is_leaf(nd):
            frames[i] = rng.standard_normal((q, k))
        else:
            transfers[i] = rng.standard_normal((k, k, 1 if i == 0 else k))
    o = (nodes, frames, transfers)
    h = ht.HTTensor(tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for _ in range(d)), ht.balanced_tree(d),
                    frames, transfers)
    red, est = ht.truncate(h, rmax, 0.0)
    ref, oest = oht.truncate(o, rmax, 0.0)
    mine = red.to_oracle()
    print((d, q, k, rmax), "ranks", red.ranks, "est", est, oest, "rel", metrics.ht_rel_diff(ref, mine),
          "norm mine", oht.norm(mine), "norm ref", oht.norm(ref), "norm in", oht.norm(o))
    for i in range(len(nodes)):
        a = mine[1][i] if mine[1][i] is not None else mine[2][i]
        print("   node", i, a.shape, float(np.abs(a).max()), float(np.isfinite(a).all()))
