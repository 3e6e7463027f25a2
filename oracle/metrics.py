"""TEST INFRASTRUCTURE ONLY -- the stable parity metric of SURVEY 8(d).

``rel(f, g) = ||f - g|| / ||f||`` computed through orthogonal transformations
only: the difference CP tensor ``add(f, scale(g, -1))`` is converted with
``from_cp`` (ht.py:165-186) and its norm taken by ``ht.norm`` (ht.py:279-282),
which orthogonalizes leaves-to-root by QR (ht.py:294-310).  Resolution ~1e-14,
unlike the Gram identity (floor ~1.5e-8).
"""

from __future__ import annotations

import numpy as np

from . import cp_als, ht_hsvd


def cp_rel_diff(f, g):
    f = [np.asarray(x) for x in f]
    g = [np.asarray(x) for x in g]
    diff = cp_als.add(f, cp_als.scale(g, -1.0))
    nf = cp_als.norm(f)
    return ht_hsvd.norm(ht_hsvd.from_cp(diff)) / (nf if nf > 0 else 1.0)


def ht_rel_diff(h1, h2):
    diff = ht_hsvd.add(h1, ht_hsvd.scale(h2, -1.0))
    n1 = ht_hsvd.norm(h1)
    return ht_hsvd.norm(diff) / (n1 if n1 > 0 else 1.0)
