"""Debug: hSVD parity over (d, Q, k) with and without the Cholesky frame factor."""
import ctypes
import math
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import ht_hsvd as oht, metrics
from paper_1803_10270_b200 import ht, _lib
from paper_1803_10270_b200.basis import BasisSpec

L = _lib.lib()
for chol in (1, 0):
    L.tp_debug_set_ht_chol(chol)
    for (d, q, k) in [(3, 7, 6), (3, 10, 8), (3, 20, 16), (3, 30, 16), (3, 30, 20), (3, 30, 24), (3, 30, 28),
                      (3, 30, 30), (3, 40, 30), (3, 40, 17), (2, 30, 30), (4, 30, 30), (5, 30, 30), (4, 40, 20),
                      (8, 20, 20)]:
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
        red, est = ht.truncate(h, k, 0.0)
        ref, oest = oht.truncate(o, k, 0.0)
        print("chol", chol, (d, q, k), "rel %.3e" % metrics.ht_rel_diff(ref, red.to_oracle()), flush=True)
L.tp_debug_set_ht_chol(1)
