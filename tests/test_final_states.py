"""CPU pins of the full-length final-state fixtures (tests/golden/final_*.npz,
written by tests/golden/make_final_states.py from the oracle).

Configs 0 and 3 are recomputed here by the oracle (seconds) and must reproduce
the committed files bitwise-closely; the config-2 file (90 min of oracle work)
is checked for shape/metadata and against a short live prefix elsewhere
(tests/test_gpu_final.py compares the GPU trajectory with it)."""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import metrics

import sys
sys.path.insert(0, str(GOLDEN))
import make_final_states as mfs  # noqa: E402


def load(part):
    z = np.load(GOLDEN / f"final_{part}.npz")
    return [z[f"f_{k}"] for k in range(int(z["d"]))], z


@pytest.mark.parametrize("which", ["cfg0", "cfg3"])
def test_explicit_fixture_reproduces(which):
    f, z = load(which)
    live = mfs.run_explicit(which, False)
    assert metrics.cp_rel_diff(f, live) <= 1e-13
    assert int(z["steps"]) == (100 if which == "cfg0" else 200)


@pytest.mark.parametrize("which,shape", [("cfg0", (32, 6)), ("cfg3", (64, 12)), ("cfg2", (128, 16))])
def test_fixture_shapes_and_sensitivity(which, shape):
    f, z = load(which)
    fp, zp = load(which + "p")
    assert len(f) == 6 and all(m.shape == shape for m in f)
    assert float(zp["perturbation"]) == 1e-13 and float(z["perturbation"]) == 0.0
    # the trajectory's own sensitivity to a 1e-13 relative input perturbation is far under the 1e-8 gate
    assert metrics.cp_rel_diff(f, fp) <= 1e-10
