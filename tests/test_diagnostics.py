"""Diagnostics.  CPU: the oracle restatement against values the
reference produced (tests/golden/diagnostics.npz).  GPU: the device contractions
(tp_cp_contract_f64) against the oracle formulas with the same weights, moments
of a sampled Maxwellian, probe evaluation against the exact function."""

import math

import numpy as np
import pytest

from conftest import load_golden, unpack_cp
from oracle import diagnostics as odiag


def test_oracle_pinned_to_reference():
    g = load_golden("diagnostics")
    assert odiag.nmae(g["nmae_x"], g["nmae_y"]) == pytest.approx(float(g["nmae"]), rel=1e-15)
    assert odiag.fit_decay_rate(g["fit_t"], g["fit_series"]) == pytest.approx(float(g["fit_rate"]), rel=1e-13)
    assert odiag.fit_decay_rate(g["fit_t"], g["fit_series"], 1e-6) == pytest.approx(float(g["fit_rate_floor"]), rel=1e-13)
    f = unpack_cp(g, "mw")
    w0, w1, w2 = (list(g[f"mw_w{p}"]) for p in (0, 1, 2))
    rho, u, T = odiag.moments(f, w0, w1, w2, float(g["mw_R"]), 1.0, [0, 1, 2])
    ref = g["mw_out"]
    assert rho == pytest.approx(ref[0], rel=1e-13)
    np.testing.assert_allclose(u, ref[1:4], atol=1e-12)
    assert T == pytest.approx(ref[4], rel=1e-12)


def test_host_functions_match_reference():
    from paper_1803_10270_b200 import diagnostics as ddiag
    g = load_golden("diagnostics")
    assert ddiag.nmae(g["nmae_x"], g["nmae_y"]) == pytest.approx(float(g["nmae"]), rel=1e-15)
    assert ddiag.fit_decay_rate(g["fit_t"], g["fit_series"], 1e-6) == pytest.approx(float(g["fit_rate_floor"]),
                                                                                    rel=1e-13)
    with pytest.raises(ValueError, match="five samples"):
        ddiag.fit_decay_rate([0, 1], [1, 2])
    with pytest.raises(ValueError, match="degenerate"):
        ddiag.nmae([1.0, 1.0], [1.0, 1.0])


@pytest.mark.gpu
def test_device_contractions_match_oracle():
    from paper_1803_10270_b200 import cp, diagnostics as ddiag
    from paper_1803_10270_b200.basis import BasisSpec, quadrature_weights
    rng = np.random.default_rng(4)
    specs = (BasisSpec(16, math.pi, "collocation", lo=0.0), BasisSpec(12, 5.0, "uniform"),
             BasisSpec(9, 5.0, "uniform"))
    f = [rng.standard_normal((s.Q, 7)) for s in specs]
    F = cp.CPTensor(specs, f)
    sets = []
    for p in (0, 1, 2):
        sets.append([quadrature_weights(s, p) for s in specs])
    got = ddiag.contract(F, np.stack([np.concatenate(ws) for ws in sets]))
    for i, ws in enumerate(sets):
        assert got[i] == pytest.approx(odiag.contract(f, ws), rel=1e-13, abs=1e-13)


@pytest.mark.gpu
def test_moments_of_sampled_maxwellian():
    from paper_1803_10270_b200 import cp, diagnostics as ddiag
    from paper_1803_10270_b200.basis import BasisSpec, nodes

    class Gas:
        R, b_x = 208.0, math.pi
    RT = Gas.R * 300.0
    bv = 8.0 * math.sqrt(RT)
    vs = BasisSpec(129, bv, "uniform")
    u0 = (0.3, -0.2, 0.1)
    cols = [np.exp(-(nodes(vs) - u0[k] * math.sqrt(RT)) ** 2 / (2 * RT))[:, None] / math.sqrt(2 * math.pi * RT)
            for k in range(3)]
    xs = BasisSpec(8, math.pi, "collocation", lo=0.0)
    f6 = cp.CPTensor((xs,) * 3 + (vs,) * 3, [np.ones((8, 1))] * 3 + cols)
    rep = ddiag.moments(f6, Gas)
    assert rep.mean_density == pytest.approx(1.0, rel=1e-6)
    np.testing.assert_allclose(rep.mean_velocity / math.sqrt(RT), u0, atol=1e-6)
    assert rep.mean_temperature == pytest.approx(300.0, rel=1e-5)
    f3 = cp.CPTensor((vs,) * 3, cols)
    assert ddiag.moments(f3, Gas).mean_temperature == pytest.approx(300.0, rel=1e-5)


@pytest.mark.gpu
def test_probe_evaluation_is_the_interpolant():
    from paper_1803_10270_b200 import cp, diagnostics as ddiag
    from paper_1803_10270_b200.basis import BasisSpec, nodes
    s = BasisSpec(24, math.pi, "collocation", lo=0.0)
    x = nodes(s)
    f = cp.CPTensor((s, s), [np.stack([np.sin(x), np.cos(2 * x)], 1), np.stack([np.cos(x), np.sin(3 * x)], 1)])
    z = np.array([[0.3, 1.7], [4.0, 2.2], [6.0, 0.1]])
    exact = np.sin(z[:, 0]) * np.cos(z[:, 1]) + np.cos(2 * z[:, 0]) * np.sin(3 * z[:, 1])
    np.testing.assert_allclose(ddiag.evaluate(f, z), exact, atol=1e-13)
    assert ddiag.evaluate(f, z[0]) == pytest.approx(exact[0], abs=1e-13)
    err = ddiag.relative_pointwise_error(lambda p, t: math.sin(p[0]) * math.cos(p[1]) + math.cos(2 * p[0]) *
                                         math.sin(3 * p[1]), f, z[1], 0.0)
    assert err < 1e-12
