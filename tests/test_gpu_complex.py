"""GPU parity of the complex128 CP path against fixtures the
reference produced in its own complex arithmetic (tests/golden/cp_als.npz
complex_*, operators.npz gal_*, complex.npz) and against the oracle."""

import numpy as np
import pytest

from conftest import load_golden, unpack_cp
from oracle import cp_als as ocp
from oracle import metrics

pytestmark = pytest.mark.gpu

from paper_1803_10270_b200 import cp, explicit, operators  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402

TOL_TRUNC = 1e-9


def crand(rng, qs, r, s=1.0):
    return [s * (rng.standard_normal((q, r)) + 1j * rng.standard_normal((q, r))) for q in qs]


def test_complex_tensor_roundtrip_and_promotion():
    rng = np.random.default_rng(0)
    S = (BasisSpec(5, 1.0), BasisSpec(7, 2.0))
    F = crand(rng, (5, 7), 3)
    T = cp.CPTensor(S, F)
    assert T.is_complex
    for a, b in zip(F, T.to_numpy()):
        np.testing.assert_array_equal(a, b)
    R = cp.CPTensor(S, [f.real.copy() for f in F])
    assert not R.is_complex
    s = cp.scale(R, 2.0 - 0.5j)                       # complex scalar promotes (cp.py:104-108)
    assert s.is_complex
    np.testing.assert_allclose(s.to_numpy()[0], (2.0 - 0.5j) * F[0].real, rtol=0, atol=1e-15)
    u = cp.add(R, T)                                   # term order: R's, then T's (cp.py:98-101)
    assert u.is_complex and u.rank == 6
    ref = ocp.add([f.real for f in F], F)
    for a, b in zip(ref, u.to_numpy()):
        np.testing.assert_array_equal(a, b)


def test_complex_inner_product_and_norm():
    rng = np.random.default_rng(1)
    qs = (6, 5, 4)
    S = tuple(BasisSpec(q, 1.0, "collocation") for q in qs)
    f, g = crand(rng, qs, 3), crand(rng, qs, 4)
    got = cp.inner_product(cp.CPTensor(S, f), cp.CPTensor(S, g))
    ref = ocp.inner_product(f, g)
    assert abs(got - ref) <= 1e-13 * abs(ref)
    # mixed real / complex promotes the real operand
    fr = [x.real.copy() for x in f]
    got2 = cp.inner_product(cp.CPTensor(S, fr), cp.CPTensor(S, g))
    assert abs(got2 - ocp.inner_product(fr, g)) <= 1e-13 * abs(ocp.inner_product(fr, g))
    assert cp.norm(cp.CPTensor(S, f)) == pytest.approx(ocp.norm(f), rel=1e-14)


def test_complex_apply_galerkin_golden():
    """operators.apply with the reference's complex Galerkin factor matrices
    (advection_operator(spiral_matrix), operators.py:65-87), against its output."""
    g = load_golden("operators")
    specs = (BasisSpec(5, 1.5), BasisSpec(7, 2.0), BasisSpec(3, 0.8))
    nt = int(g["gal_nterms"])
    rows = tuple(tuple(g[f"gal_E{t}_{k}"] if f"gal_E{t}_{k}" in g else None for k in range(3)) for t in range(nt))
    op = operators.SeparableOperator(specs, tuple(complex(w) for w in g["gal_weights"]), rows)
    out = operators.apply(op, cp.CPTensor(specs, unpack_cp(g, "gal_f")))
    assert out.is_complex
    for a, b in zip(unpack_cp(g, "gal_out"), out.to_numpy()):
        np.testing.assert_allclose(b, a, rtol=0, atol=1e-13 * np.abs(a).max())


def test_complex_als_reference_golden():
    """cp_approx_als in the reference's native complex arithmetic: trace-scaled
    lambda, default stall rule (cp.py:166-180, 329-332), 40-sweep cap."""
    g = load_golden("cp_als")
    V, init = unpack_cp(g, "complex_V"), unpack_cp(g, "complex_init")
    S = (BasisSpec(5, np.pi), BasisSpec(7, np.pi), BasisSpec(3, np.pi))
    trace = []
    out = cp.cp_approx_als(cp.CPTensor(S, V), 2, cp.ALSApproxConfig(max_sweeps=40), init=cp.CPTensor(S, init),
                           trace=trace)
    assert out.is_complex
    assert metrics.cp_rel_diff(unpack_cp(g, "complex_out"), out.to_numpy()) <= TOL_TRUNC
    gt = g["complex_trace"]
    n = min(len(trace), len(gt))
    assert abs(len(trace) - len(gt)) <= 1
    np.testing.assert_allclose(trace[:n], gt[:n], rtol=1e-7, atol=1e-12)


@pytest.mark.parametrize("qs,R,r,lam", [((9, 9), 12, 3, 1e-10), ((5, 7, 3), 8, 4, None), ((11, 6, 8, 5), 20, 6, 1e-10),
                                        ((33, 17, 9), 40, 8, None)])
def test_complex_als_vs_oracle(qs, R, r, lam):
    rng = np.random.default_rng(R + r)
    S = tuple(BasisSpec(q, 1.0, "collocation") for q in qs)
    V = crand(rng, qs, R, 0.3)
    init = [v[:, :r].copy() for v in V]
    sweeps = 12
    trace, otrace = [], []
    out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=lam),
                           init=cp.CPTensor(S, init), trace=trace)
    ref = ocp.als(V, init, sweeps, lam=lam, stall=-np.inf, trace=otrace)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    np.testing.assert_allclose(trace, otrace, rtol=1e-8, atol=1e-12)


def test_complex_als_default_init_is_reference_draw():
    """Without init, the guess is the reference's seeded complex random_cp (cp.py:300-301)."""
    rng = np.random.default_rng(3)
    qs = (5, 7)
    S = tuple(BasisSpec(q, 1.0) for q in qs)
    V = crand(rng, qs, 5, 0.4)
    out = cp.cp_approx_als(cp.CPTensor(S, V), 2, cp.ALSApproxConfig(max_sweeps=6, stall=-np.inf, seed=4))
    init = ocp.random_cp(list(qs), 2, np.random.default_rng(4))
    ref = ocp.als(V, init, 6, lam=None, stall=-np.inf)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC


def test_complex_rank_reduce_golden():
    """rank_reduce_als with the reference's complex random terms (cp.py:337-366).
    The fits stop on the stall rule (1e-13 ||t|| per sweep) of a linearly
    converging ALS, so two correct implementations that round differently stop
    ~1e-8 apart along the convergence path: the gate is the reference's own
    distance to the exact rank-2 target (+50%), and 2e-8 to the reference fit."""
    g = load_golden("complex")
    S = (BasisSpec(5, 1.5), BasisSpec(7, 2.0), BasisSpec(3, 0.8))
    f = unpack_cp(g, "rr_f")
    out = cp.rank_reduce_als(cp.CPTensor(S, f), 3, 1e-9)
    gold = unpack_cp(g, "rr_out")
    assert out.rank == gold[0].shape[1]
    got = out.to_numpy()
    assert metrics.cp_rel_diff(f, got) <= 1.5 * metrics.cp_rel_diff(f, gold) + 1e-12
    assert metrics.cp_rel_diff(gold, got) <= 2e-8


def test_rank_reduce_reference_draws_real_target_golden():
    """rank_reduce_als(..., draws="reference") on a REAL target: the reference's complex
    random terms (cp.py:356-360), so the fit is complex like the reference's; pinned to
    the reference's own output (tests/golden/make_golden.py gen_complex, rrr_*)."""
    g = load_golden("complex")
    S = (BasisSpec(5, 1.5), BasisSpec(7, 2.0), BasisSpec(3, 0.8))
    f = unpack_cp(g, "rrr_f")
    assert not any(np.iscomplexobj(x) and np.any(x.imag) for x in f)
    out = cp.rank_reduce_als(cp.CPTensor(S, f), 3, 1e-9, draws="reference")
    gold = unpack_cp(g, "rrr_out")
    assert out.is_complex and out.rank == gold[0].shape[1]
    got = out.to_numpy()
    assert metrics.cp_rel_diff(f, got) <= 1.5 * metrics.cp_rel_diff(f, gold) + 1e-12
    assert metrics.cp_rel_diff(gold, got) <= 2e-8
    with pytest.raises(ValueError, match="draws"):
        cp.rank_reduce_als(cp.CPTensor(S, f), 3, 1e-9, draws="nope")


def test_complex_explicit_split_recipe_golden():
    """The reference's explicit recipe (explicit.py:85-103, rank_reduce_als at every
    stage) on the complex Galerkin basis, 2-D sheared advection, RK2 + 2 AB2 steps."""
    g = load_golden("complex")
    q, b, dt, r_max, eps = g["ex_meta"]
    S = (BasisSpec(int(q), float(b)), BasisSpec(int(q), float(b)))
    nt = int(g["ex_nterms"])
    rows = tuple(tuple(g[f"ex_E{t}_{k}"] if f"ex_E{t}_{k}" in g else None for k in range(2)) for t in range(nt))
    op = operators.SeparableOperator(S, tuple(complex(w) for w in g["ex_weights"]), rows)
    cfg = explicit.ExplicitConfig(dt=float(dt), r_max=int(r_max), eps_rank=float(eps), recipe="split")
    f0 = cp.CPTensor(S, unpack_cp(g, "ex_step0"))
    traj = [f0, explicit.startup_step(f0, op, cfg)]
    for _ in range(2):
        traj.append(explicit.ab2_step(traj[-2], traj[-1], op, cfg))
    for n, f in enumerate(traj):
        assert metrics.cp_rel_diff(unpack_cp(g, f"ex_step{n}"), f.to_numpy()) <= 1e-8, n
