"""GPU parity: CP inner products, operator apply and the fused ALS kernel vs the
oracle (oracle/ is pinned to the reference by tests/golden).  Bar: the stable
relative difference of represented tensors <= 1e-9 per truncation (BASELINE
north star); inner products to 1e-12 relative."""

import math

import numpy as np
import pytest
import torch

from conftest import load_golden, unpack_cp
from oracle import cp_als as ocp
from oracle import metrics, operators as oops

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_1803_10270_b200")
from paper_1803_10270_b200 import cp, operators, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec  # noqa: E402

TOL_TRUNC = 1e-9


def specs_for(qs):
    return tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for q in qs)


def rand_factors(rng, qs, r, scale=1.0):
    return [scale * rng.standard_normal((q, r)) for q in qs]


@pytest.mark.parametrize("qs,ra,rb", [((5, 7, 3), 3, 4), ((16,) * 6, 40, 40), ((33, 17, 64, 8), 70, 5),
                                       ((256,) * 6, 512, 512), ((1, 2, 3), 1, 1)])
def test_inner_product_matches_oracle(qs, ra, rb):
    rng = np.random.default_rng(ra * 1000 + rb)
    f = rand_factors(rng, qs, ra, 1 / math.sqrt(max(qs)))
    g = rand_factors(rng, qs, rb, 1 / math.sqrt(max(qs)))
    S = specs_for(qs)
    F, G = cp.CPTensor(S, f), cp.CPTensor(S, g)
    ref = ocp.inner_product(f, g).real
    got = cp.inner_product(F, G)
    assert abs(got - ref) <= 1e-12 * max(abs(ref), 1e-300) + 1e-14 * math.sqrt(abs(ocp.inner_product(f, f).real * ocp.inner_product(g, g).real))
    # symmetric path (same buffer, upper tiles only)
    ref_ff = ocp.inner_product(f, f).real
    assert abs(cp.inner_product(F, F) - ref_ff) <= 1e-12 * abs(ref_ff)
    assert abs(cp.norm(F) - math.sqrt(ref_ff)) <= 1e-12 * math.sqrt(ref_ff)


def test_apply_matches_oracle():
    g = load_golden("operators")
    fr = unpack_cp(g, "col_f")
    D, a = g["col_D"], g["col_a"]
    S = specs_for([D.shape[0]] * 3)
    op = operators.SeparableOperator(S, tuple(-a), tuple(tuple(D if k == t else None for k in range(3))
                                                       for t in range(3)))
    out = operators.apply(op, cp.CPTensor(S, fr))
    ref = unpack_cp(g, "col_out")
    for x, y in zip(out.to_numpy(), ref):
        np.testing.assert_allclose(x, y, rtol=0, atol=1e-13)


def test_add_scale_concatenate():
    rng = np.random.default_rng(3)
    S = specs_for((6, 5, 4))
    f, g = rand_factors(rng, (6, 5, 4), 2), rand_factors(rng, (6, 5, 4), 3)
    s = cp.add(cp.CPTensor(S, f), cp.scale(cp.CPTensor(S, g), -2.5))
    ref = ocp.add(f, ocp.scale(g, -2.5))
    assert s.rank == 5
    for x, y in zip(s.to_numpy(), ref):
        np.testing.assert_array_equal(x, y)


def _als_case(V, init, sweeps, lam, stall=-np.inf, grid=0):
    qs = [v.shape[0] for v in V]
    S = specs_for(qs)
    T = cp.CPTensor(S, V)
    I0 = cp.CPTensor(S, init)
    trace = []
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, tol=0.0, stall=stall, reg=lam, grid=grid)
    out = cp.cp_approx_als(T, init[0].shape[1], cfg, init=I0, trace=trace)
    otrace = []
    ref = ocp.als(V, init, sweeps, lam=lam, stall=stall, trace=otrace)
    return out, ref, trace, otrace


def test_als_golden_cases():
    g = load_golden("cp_als")
    for name in g["names"]:
        name = str(name)
        V = unpack_cp(g, f"{name}_V")
        init = unpack_cp(g, f"{name}_init")
        sweeps, lam, stall, r = g[f"{name}_meta"]
        out, ref, trace, otrace = _als_case(V, init, int(sweeps), None if lam < 0 else float(lam), stall)
        gold = unpack_cp(g, f"{name}_out")
        rel = metrics.cp_rel_diff(gold, out.to_numpy())
        assert rel <= TOL_TRUNC, (name, rel)
        assert len(trace) == len(g[f"{name}_trace"]), name
        np.testing.assert_allclose(trace, g[f"{name}_trace"], rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("grid", [0, 1, 3, 17])
def test_als_grid_sizes(grid):
    rng = np.random.default_rng(7)
    qs, R, r = (20, 24, 16, 12, 9), 37, 5
    V = rand_factors(rng, qs, R, 0.3)
    init = [v[:, :r].copy() for v in V]
    out, ref, trace, otrace = _als_case(V, init, 12, 1e-10, grid=grid)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-10)


@pytest.mark.parametrize("r", [1, 6, 12, 16, 31, 32])
def test_als_ranks(r):
    rng = np.random.default_rng(100 + r)
    qs, R = (24,) * 4, 3 * r + 5
    V = rand_factors(rng, qs, R, 0.2)
    init = [v[:, :r].copy() for v in V]
    out, ref, _, _ = _als_case(V, init, 8, 1e-10)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC


def test_als_config1_full_size():
    w = workloads.cfg1(seed=0)
    out, ref, trace, otrace = _als_case(w["V"], w["init"], w["sweeps"], w["lam"])
    rel = metrics.cp_rel_diff(ref, out.to_numpy())
    assert rel <= TOL_TRUNC, rel
    assert len(trace) == 20
    np.testing.assert_allclose(trace, otrace, rtol=1e-9)


def test_als_deterministic_bitwise():
    w = workloads.cfg1(seed=1, Q=64, R=128, r=16)
    S = specs_for([64] * 6)
    T, I0 = cp.CPTensor(S, w["V"]), cp.CPTensor(S, w["init"])
    cfg = cp.ALSApproxConfig(max_sweeps=5, stall=-np.inf, reg=1e-10)
    a = cp.cp_approx_als(T, 16, cfg, init=I0)
    b = cp.cp_approx_als(T, 16, cfg, init=I0)
    assert torch.equal(a.data, b.data)


def test_als_stall_stop_matches_reference_rule():
    rng = np.random.default_rng(9)
    qs, r = (9, 8, 7, 6), 3
    V = rand_factors(rng, qs, 10)
    init = [v[:, :r].copy() for v in V]
    out, ref, trace, otrace = _als_case(V, init, 200, None, stall=1e-13)
    assert len(trace) == len(otrace)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC


def test_als_zero_sweeps_returns_init_copy():
    rng = np.random.default_rng(5)
    S = specs_for((5, 6))
    V = cp.CPTensor(S, rand_factors(rng, (5, 6), 4))
    I0 = cp.CPTensor(S, rand_factors(rng, (5, 6), 2))
    out = cp.cp_approx_als(V, 2, cp.ALSApproxConfig(max_sweeps=0), init=I0)
    assert torch.equal(out.data, I0.data) and out.data.data_ptr() != I0.data.data_ptr()


def test_als_rejects_bad_init():
    rng = np.random.default_rng(5)
    S = specs_for((5, 6))
    V = cp.CPTensor(S, rand_factors(rng, (5, 6), 4))
    with pytest.raises(ValueError, match="init"):
        cp.cp_approx_als(V, 2, init=cp.CPTensor(S, rand_factors(rng, (5, 6), 3)))
    with pytest.raises(ValueError, match="specs"):
        cp.cp_approx_als(lambda p: p, 2)


def test_rank_reduce_strips_noise():
    rng = np.random.default_rng(8)
    S = specs_for((7, 6, 5))
    clean = cp.CPTensor(S, rand_factors(rng, (7, 6, 5), 2))
    noisy = cp.pad_rank(clean, 4, rng, rel_scale=1e-9)
    red = cp.rank_reduce_als(noisy, 2, eps=1e-7)
    assert red.rank <= 2
    rel = metrics.cp_rel_diff(noisy.to_numpy(), red.to_numpy())
    assert rel < 1e-7


@pytest.fixture
def als_variant():
    """Force the ALS kernel variant through the library's debug hook, restore auto after."""
    import ctypes
    from paper_1803_10270_b200 import _lib
    L = _lib.lib()
    L.tp_debug_set_als_variant.argtypes = [ctypes.c_int, ctypes.c_int]

    def set_(variant, cluster=0):
        L.tp_debug_set_als_variant(variant, cluster)
    yield set_
    L.tp_debug_set_als_variant(0, 0)


@pytest.mark.parametrize("variant,cluster", [(1, 0), (2, 2), (2, 4), (2, 0), (4, 0), (8, 16), (8, 8)])
@pytest.mark.parametrize("qs,R,r", [((64, 48, 80, 64), 96, 16), ((40, 37, 50), 61, 12), ((32,) * 5, 64, 30)])
def test_als_kernel_variants(als_variant, variant, cluster, qs, R, r):
    """Both persistent kernels (R-slab per CTA; clusters of row blocks with the DSMEM
    cross all-reduce; variant 4 = the R-slab kernel as ONE cluster with hardware
    cluster barriers) on ragged mode sizes / slab widths, with the residual trace."""
    als_variant(variant, cluster)
    rng = np.random.default_rng(R + r)
    V = rand_factors(rng, qs, R, 0.25)
    init = [v[:, :r].copy() for v in V]
    out, ref, trace, otrace = _als_case(V, init, 9, 1e-10)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    np.testing.assert_allclose(trace, otrace, rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("variant,cluster", [(1, 0), (2, 4), (8, 16)])
def test_als_config1_variants(als_variant, variant, cluster):
    als_variant(variant, cluster)
    w = workloads.cfg1(seed=2)
    out, ref, _, _ = _als_case(w["V"], w["init"], w["sweeps"], w["lam"])
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC


def test_als_deferred_check_matches_sync():
    rng = np.random.default_rng(12)
    qs, R, r = (12, 10, 14), 20, 4
    S = specs_for(qs)
    V = cp.CPTensor(S, rand_factors(rng, qs, R, 0.3))
    I0 = cp.CPTensor(S, [f[:, :r].copy() for f in V.to_numpy()])
    cfg = cp.ALSApproxConfig(max_sweeps=6, stall=-np.inf, reg=1e-10)
    a = cp.cp_approx_als(V, r, cfg, init=I0)
    b = cp.check(cp.cp_approx_als(V, r, cfg, init=I0, sync=False))
    assert torch.equal(a.data, b.data) and b.pending_info is None
    with pytest.raises(ValueError, match="trace"):
        cp.cp_approx_als(V, r, cfg, init=I0, sync=False, trace=[])


@pytest.mark.parametrize("qs,R,r", [((32,) * 6, 78, 6), ((5, 7, 3), 6, 2), ((9, 8, 7, 6), 10, 3), ((20, 16, 24), 41, 12),
                                    ((16, 12), 40, 9)])
def test_als_small_variant(als_variant, qs, R, r):
    """One CTA with the whole problem in shared memory (config 0 sizes and ragged
    shapes), with the residual trace; forced through the debug hook."""
    als_variant(3, 0)
    rng = np.random.default_rng(R + 7 * r)
    V = rand_factors(rng, qs, R, 0.3)
    init = [v[:, :r].copy() for v in V]
    out, ref, trace, otrace = _als_case(V, init, 10, 1e-10)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    np.testing.assert_allclose(trace, otrace, rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("qs,R,r", [((32,) * 6, 78, 6), ((5, 7, 3), 6, 2), ((9, 8, 7, 6), 10, 3), ((20, 16, 24), 41, 8),
                                    ((16, 12), 40, 1), ((33, 17, 40, 9, 12), 29, 7)])
def test_als_tiny8_variant(als_variant, qs, R, r):
    """r <= 8 in one CTA on the DMMA pipe (zero-padded tiles: ragged Q, R not a
    multiple of 8), with the residual trace; forced through the debug hook."""
    als_variant(5, 0)
    rng = np.random.default_rng(R + 11 * r)
    V = rand_factors(rng, qs, R, 0.3)
    init = [v[:, :r].copy() for v in V]
    out, ref, trace, otrace = _als_case(V, init, 10, 1e-10)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    np.testing.assert_allclose(trace, otrace, rtol=1e-8, atol=1e-12)


def test_als_auto_plan_config0_is_tiny8():
    from paper_1803_10270_b200 import cp as _cp
    assert _cp.als_plan((32,) * 6, 78, 6)["kernel"] == "als_tiny8"


@pytest.mark.parametrize("early", [0, 1])
@pytest.mark.parametrize("variant", [1, 4])
def test_als_early_inverse_toggle(als_variant, variant, early):
    """r <= 16 multi-CTA truncations with the exact inverse formed in phase A by warps
    0-3 (default) and with the phase-B Newton-Schulz / exact solve (debug hook off)."""
    import ctypes
    from paper_1803_10270_b200 import _lib
    L = _lib.lib()
    L.tp_debug_set_als_early_inv.argtypes = [ctypes.c_int]
    als_variant(variant, 0)
    L.tp_debug_set_als_early_inv(early)
    try:
        rng = np.random.default_rng(40 + early)
        qs, R, r = (64, 48, 33, 64, 20), 150, 12
        V = rand_factors(rng, qs, R, 0.25)
        init = [v[:, :r].copy() for v in V]
        out, ref, trace, otrace = _als_case(V, init, 8, 1e-10)
        assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
        np.testing.assert_allclose(trace, otrace, rtol=1e-8, atol=1e-12)
    finally:
        L.tp_debug_set_als_early_inv(1)


@pytest.mark.parametrize("qs,R,r", [((7,), 5, 2), ((9, 1), 4, 1), ((1, 1, 1), 3, 1), ((6, 5), 1, 1), ((8, 7, 6), 3, 5),
                                    ((2, 3, 2, 3, 2, 3, 2, 3), 4, 3)])
def test_als_edge_shapes(qs, R, r):
    """Degenerate shapes the reference accepts: one mode, Q = 1 modes, rank-1 targets,
    r > R (rank-deficient normal equations held by lambda), d = 8 (TP_MAXD).  (A Q = 1
    mode with r > 1 makes the normal equations rank-deficient up to lambda: the fit is
    then conditioned ~1/lambda and differs from the oracle at that level.)"""
    rng = np.random.default_rng(len(qs) * 10 + R + r)
    V = rand_factors(rng, qs, R, 0.5)
    init = [rng.standard_normal((q, r)) * 0.3 for q in qs]
    out, ref, trace, otrace = _als_case(V, init, 6, 1e-6)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    # residual trace by the Gram identity: absolute floor ~sqrt(eps) ||V||
    np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-8 * max(1.0, float(np.sqrt(sum(
        np.sum(v * v) for v in V)))))


def test_als_rejects_bad_shapes():
    rng = np.random.default_rng(0)
    S = specs_for((4, 5))
    T = cp.CPTensor(S, rand_factors(rng, (4, 5), 6, 0.5))
    with pytest.raises(ValueError, match="init shape"):
        cp.cp_approx_als(T, 3, cp.ALSApproxConfig(max_sweeps=2), init=cp.CPTensor(S, rand_factors(rng, (4, 5), 2, 1.0)))
    with pytest.raises(ValueError):
        cp.cp_approx_als(T, 200, cp.ALSApproxConfig(max_sweeps=2))   # r > 160: outside every variant


@pytest.mark.parametrize("variant,cluster", [(0, 0), (1, 0), (2, 0), (3, 0), (4, 0), (5, 0), (8, 0)])
@pytest.mark.parametrize("reg", [None, 1e-10])
def test_als_zero_target_returns_zero(als_variant, variant, cluster, reg):
    """All-zero target: under the reference trace rule lambda = 1e-12 tr(H)/r is 0 once a
    factor is zero, np.linalg.solve raises LinAlgError and _solve_gram falls back to lstsq
    (cp.py:176-177), whose min-norm solution is 0 -- the fit is all zeros, not an error
    (ADVICE r1).  Every kernel variant; fixed lambda likewise."""
    als_variant(variant, cluster)
    rng = np.random.default_rng(9)
    qs, R, r = (12, 9, 10, 8), 10, 6
    S = specs_for(qs)
    T = cp.CPTensor(S, [np.zeros((q, R)) for q in qs])
    init = cp.CPTensor(S, rand_factors(rng, qs, r, 0.5))
    cfg = cp.ALSApproxConfig(max_sweeps=3, stall=-np.inf, reg=reg, grid=2 if variant == 4 else 0)
    out = cp.cp_approx_als(T, r, cfg, init=init)
    assert torch.count_nonzero(out.data).item() == 0
    # complex128 path (one-CTA complex kernel) follows the same rule
    if variant == 0:
        Tc = cp.as_complex(T)
        outc = cp.cp_approx_als(Tc, r, cp.ALSApproxConfig(max_sweeps=3, stall=-np.inf, reg=reg),
                                init=cp.as_complex(init))
        assert torch.count_nonzero(outc.data).item() == 0


# ---- streamed generic variant (r > 32, targets beyond shared memory) ----------------

@pytest.mark.parametrize("r,R,sweeps", [(40, 4096, 3), (64, 4096, 2)])
def test_als_generic_large_rank_and_input(r, R, sweeps):
    """r = 40 / 64 and R = 4096 at Q = 256, d = 6 (beyond the fused kernels' r <= 32 and
    their aggregate-shared-memory limit): the streamed variant, oracle parity <= 1e-9."""
    qs = (256,) * 6
    assert cp.als_plan(qs, R, r)["kernel"] == "als_generic"
    rng = np.random.default_rng(r + R)
    V = [rng.standard_normal((q, R)) / 16 for q in qs]
    init = [v[:, :r].copy() for v in V]
    out = cp.cp_approx_als(cp.CPTensor(specs_for(qs), V), r,
                           cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10),
                           init=cp.CPTensor(specs_for(qs), init))
    ref = ocp.als(V, init, sweeps, lam=1e-10)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC


def test_als_fused_limit_large_R_streams():
    """R = 4096 with r = 32 no longer fits the fused kernels' shared memory: the plan
    falls back to the streamed variant instead of raising."""
    assert cp.als_plan((256,) * 6, 4096, 32)["kernel"] == "als_generic"


@pytest.mark.parametrize("reg", [1e-10, None])
@pytest.mark.parametrize("qs,R,r", [((12, 9, 10, 8), 30, 7), ((20, 16, 24), 50, 33), ((16,) * 5, 40, 48)])
def test_als_generic_forced_matches_oracle(als_variant, qs, R, r, reg):
    """The generic variant forced (debug hook 7) on small shapes, both regulariser
    rules, with the residual trace (device-side Gram identity)."""
    als_variant(7, 0)
    rng = np.random.default_rng(R + r)
    V = rand_factors(rng, qs, R, 0.3)
    init = [rng.standard_normal((q, r)) * 0.3 for q in qs]
    S = specs_for(qs)
    trace = []
    cfg = cp.ALSApproxConfig(max_sweeps=6, stall=-np.inf, reg=reg)
    out = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init), trace=trace)
    otrace = []
    ref = ocp.als(V, init, 6, lam=reg, trace=otrace)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-8)
    assert len(trace) == 6


def test_als_generic_stall_and_zero_target(als_variant):
    """Stopping rules decided on the device (cp.py:329-332): the generic variant stops
    at the same sweep as the fused kernels; an all-zero target gives a zero fit."""
    rng = np.random.default_rng(5)
    qs, R, r = (14, 12, 10), 20, 3
    S = specs_for(qs)
    V = rand_factors(rng, qs, R, 0.5)
    init = [v[:, :r].copy() for v in V]
    cfg = cp.ALSApproxConfig(max_sweeps=200, stall=1e-6, reg=1e-10)
    t_fused, t_gen = [], []
    a = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init), trace=t_fused)
    als_variant(7, 0)
    b = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init), trace=t_gen)
    assert len(t_fused) == len(t_gen) < 200
    assert metrics.cp_rel_diff(a.to_numpy(), b.to_numpy()) <= 1e-9
    Z = cp.CPTensor(S, [np.zeros((q, R)) for q in qs])
    z = cp.cp_approx_als(Z, r, cp.ALSApproxConfig(max_sweeps=3, stall=-np.inf), init=cp.CPTensor(S, init))
    assert torch.count_nonzero(z.data).item() == 0


@pytest.mark.parametrize("cplx", [False, True])
def test_apply_more_than_64_terms(cplx):
    """Operators with more terms than one kernel argument block holds (100 > 64):
    consecutive launches, same term-major output (operators.py:48-62)."""
    rng = np.random.default_rng(77)
    qs, r, nt = (6, 5, 7), 2, 100
    S = specs_for(qs)
    mats = [[rng.standard_normal((q, q)) if (t + k) % 3 == 0 else None for k, q in enumerate(qs)] for t in range(nt)]
    w = list(rng.standard_normal(nt))
    if cplx:
        w = [x + 0.5j * x for x in w]
    L = operators.SeparableOperator(S, tuple(w), tuple(tuple(m) for m in mats))
    f = rand_factors(rng, qs, r, 1.0)
    out = operators.apply(L, cp.CPTensor(S, f))
    ref = oops.apply(w, mats, [x.astype(np.complex128) if cplx else x for x in f])
    assert out.rank == nt * r
    got = out.to_numpy()
    for k in range(len(qs)):
        np.testing.assert_allclose(got[k], ref[k], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("comm", ["mc", "dsmem", "mc-unsplit"])
@pytest.mark.parametrize("ns", [6, 0])
@pytest.mark.parametrize("reg", [None, 1e-10])
@pytest.mark.parametrize("qs,R,r", [((256,) * 6, 512, 32), ((48, 40, 64, 36), 200, 16), ((20, 33, 17, 40), 64, 8)])
def test_als_rows_kernel(als_variant, comm, ns, reg, qs, R, r):
    """Cluster-row kernel (variant 8: 16-CTA clusters own R-slabs, one flag exchange per mode
    update): warm-started Newton-Schulz inverse on and off (exact sweep every time), both
    regulariser rules, ragged modes, config-1 size, with the residual trace; cluster publishes
    by TMA multicast or st.async; the rhs product beside the inverse (split warps, default)
    or before it."""
    import ctypes
    from paper_1803_10270_b200 import _lib
    L = _lib.lib()
    L.tp_debug_set_als_ns.argtypes = [ctypes.c_int]
    als_variant(8, 0)
    L.tp_debug_set_als_ns(ns)
    L.tp_debug_set_als_rows_mc.argtypes = [ctypes.c_int]
    L.tp_debug_set_als_rows_mc(0 if comm == "dsmem" else 1)    # cluster publishes: TMA multicast / st.async
    L.tp_debug_set_als_rows_split.argtypes = [ctypes.c_int]
    L.tp_debug_set_als_rows_split(0 if comm == "mc-unsplit" else 1)
    try:
        assert cp.als_plan(qs, R, r)["kernel"] == "als_rows"
        rng = np.random.default_rng(R + r + ns)
        V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
        init = [v[:, :r].copy() for v in V]
        S = specs_for(qs)
        trace = []
        out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=6, stall=-np.inf, reg=reg),
                               init=cp.CPTensor(S, init), trace=trace)
        otrace = []
        ref = ocp.als(V, init, 6, lam=reg, trace=otrace)
        assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
        np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-8 * max(1.0, float(np.sqrt(sum(
            np.sum(v * v) for v in V)))))
    finally:
        L.tp_debug_set_als_ns(6)
        L.tp_debug_set_als_rows_mc(1)
        L.tp_debug_set_als_rows_split(1)


def test_als_w_is_config1_default(als_variant):
    """Config 1 runs the Gram-space kernel (variant 9); with it disabled (debug hook) the
    cluster-row kernel is the plan again."""
    import ctypes
    from paper_1803_10270_b200 import _lib
    L = _lib.lib()
    L.tp_debug_set_als_w.argtypes = [ctypes.c_int, ctypes.c_double]
    assert cp.als_plan((256,) * 6, 512, 32)["kernel"] == "als_w"
    L.tp_debug_set_als_w(0, 0.0)
    try:
        assert cp.als_plan((256,) * 6, 512, 32)["kernel"] == "als_rows"
    finally:
        L.tp_debug_set_als_w(1, 0.0)


@pytest.mark.parametrize("reg", [None, 1e-10])
@pytest.mark.parametrize("qs,R,r", [((256,) * 6, 512, 32), ((300, 280), 1000, 32), ((200, 180, 220, 190), 515, 20),
                                    ((128, 160, 144), 259, 7), ((96,) * 6, 300, 32)])
def test_als_w_kernel(als_variant, reg, qs, R, r):
    """Gram-space kernel (variant 9): the sweeps run on the crosses / Grams with W_k = V_k^T V_k,
    U_k formed after the last sweep.  Config-1 size, ragged modes, R not a multiple of the
    8-term slab, ranks that are not tile multiples, both regulariser rules, with the residual
    trace (Gram identity, cp.py:321-326) -- against the oracle."""
    als_variant(9, 0)
    assert cp.als_plan(qs, R, r)["kernel"] == "als_w"
    rng = np.random.default_rng(R + r)
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    S = specs_for(qs)
    trace, otrace = [], []
    out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=5, stall=-np.inf, reg=reg),
                           init=cp.CPTensor(S, init), trace=trace)
    ref = ocp.als(V, init, 5, lam=reg, trace=otrace)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    tnorm = float(np.sqrt(ocp.inner_product(V, V).real))
    np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-8 * max(1.0, tnorm))
    # bitwise reproducible (fixed summation orders, data-carried synchronisation)
    again = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=5, stall=-np.inf, reg=reg),
                             init=cp.CPTensor(S, init))
    assert torch.equal(out.data, again.data)


@pytest.mark.parametrize("qs,R,r,sweeps", [((160, 144), 512, 32, 4),            # two modes (slot reuse every round)
                                           ((72,) * 7, 264, 12, 3),           # seven modes (shared memory near the limit)
                                           ((80, 96, 72), 257, 1, 3),         # rank 1, last slab one column wide
                                           ((128, 96, 112), 384, 9, 1),       # one sweep: exact inverses only
                                           ((128, 96, 112), 384, 31, 2),      # r = 31 (padded to 32)
                                           ((300, 320, 310), 1184, 16, 2)])   # one CTA per SM (148 slabs)
def test_als_w_edge_shapes(als_variant, qs, R, r, sweeps):
    """Corner shapes of the Gram-space kernel against the oracle, with the residual trace."""
    als_variant(9, 0)
    assert cp.als_plan(qs, R, r)["kernel"] == "als_w"
    rng = np.random.default_rng(7 * R + r)
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    S = specs_for(qs)
    trace, otrace = [], []
    out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10),
                           init=cp.CPTensor(S, init), trace=trace)
    ref = ocp.als(V, init, sweeps, lam=1e-10, trace=otrace)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    tnorm = float(np.sqrt(ocp.inner_product(V, V).real))
    np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-8 * max(1.0, tnorm))
    # without the trace (no residual rounds, no trailing barriers): the same fit bitwise
    out2 = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=sweeps, stall=-np.inf, reg=1e-10),
                            init=cp.CPTensor(S, init))
    assert torch.equal(out.data, out2.data)


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("qs,R,r", [((256,) * 6, 512, 32), ((200, 180, 220, 190), 515, 20), ((128, 160, 144), 259, 7)])
def test_als_w_cta_pairs(als_variant, pair, qs, R, r):
    """The K range of a column slab's T product split over a CTA pair (2-CTA clusters, partials exchanged
    through distributed shared memory) or kept in one CTA: both against the oracle, odd slab counts included."""
    import ctypes
    from paper_1803_10270_b200 import _lib
    L = _lib.lib()
    L.tp_debug_set_als_w_pair.argtypes = [ctypes.c_int]
    als_variant(9, 0)
    L.tp_debug_set_als_w_pair(pair)
    try:
        plan = cp.als_plan(qs, R, r)
        assert plan["kernel"] == "als_w" and plan["cluster"] == 1 + pair and plan["ctas"] == ((R + 7) // 8) * (1 + pair)
        rng = np.random.default_rng(R + r + pair)
        V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
        init = [v[:, :r].copy() for v in V]
        S = specs_for(qs)
        trace, otrace = [], []
        out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=4, stall=-np.inf, reg=1e-10),
                               init=cp.CPTensor(S, init), trace=trace)
        ref = ocp.als(V, init, 4, lam=1e-10, trace=otrace)
        assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
        tnorm = float(np.sqrt(ocp.inner_product(V, V).real))
        np.testing.assert_allclose(trace, otrace, rtol=1e-7, atol=1e-8 * max(1.0, tnorm))
    finally:
        L.tp_debug_set_als_w_pair(1)


def test_als_w_unsupported_shapes_fall_through(als_variant):
    """Shapes outside the Gram-space kernel's plan (eight modes: shared memory; R > 4 min Q: more work
    than the direct form; fewer than 32 slabs) keep their direct kernels in the automatic plan."""
    assert cp.als_plan((128,) * 8, 512, 32)["kernel"] != "als_w"
    assert cp.als_plan((64,) * 6, 588, 12)["kernel"] != "als_w"
    assert cp.als_plan((256,) * 4, 200, 32)["kernel"] != "als_w"


def test_als_w_tol_stop(als_variant):
    """tol rule (cp.py:329): stop after the first sweep whose residual is <= tol ||V||."""
    als_variant(9, 0)
    qs, R, r = (128,) * 4, 256, 16
    rng = np.random.default_rng(41)
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    S = specs_for(qs)
    trace, otrace = [], []
    out = cp.cp_approx_als(cp.CPTensor(S, V), r, cp.ALSApproxConfig(max_sweeps=20, tol=0.999, stall=-np.inf, reg=1e-10),
                           init=cp.CPTensor(S, init), trace=trace)
    ref = ocp.als(V, init, len(trace), lam=1e-10, trace=otrace)
    tnorm = float(np.sqrt(ocp.inner_product(V, V).real))
    assert 1 <= len(trace) < 20 and trace[-1] <= 0.999 * tnorm and all(t > 0.999 * tnorm for t in trace[:-1])
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC


def test_als_w_stopping_rules(als_variant):
    """tol / stall decided on the device after each sweep (cp.py:329-332): same sweep count as the
    oracle and as the cluster-row kernel, same fit."""
    qs, R, r = (128,) * 4, 256, 8
    rng = np.random.default_rng(17)
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    S = specs_for(qs)
    cfg = cp.ALSApproxConfig(max_sweeps=60, stall=1e-7, reg=1e-10)
    traces = {}
    outs = {}
    for variant in (8, 9):
        als_variant(variant, 0)
        assert cp.als_plan(qs, R, r)["kernel"] == {8: "als_rows", 9: "als_w"}[variant]
        traces[variant] = []
        outs[variant] = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init), trace=traces[variant])
    assert len(traces[8]) == len(traces[9]) < 60
    np.testing.assert_allclose(traces[9], traces[8], rtol=1e-9)
    assert metrics.cp_rel_diff(outs[8].to_numpy(), outs[9].to_numpy()) <= TOL_TRUNC


def test_als_w_ill_conditioned_falls_back(als_variant):
    """The Gram-space form loses ~eps cond(A_j): above the pivot-ratio bound the kernel writes
    nothing and the cluster-row kernel launched behind it reruns the truncation -- the result is
    bitwise the cluster-row kernel's own, and matches the oracle within the problem's sensitivity."""
    qs, R, r = (128,) * 4, 512, 8
    rng = np.random.default_rng(23)
    V = [rng.standard_normal((q, R)) / np.sqrt(q) for q in qs]
    init = [v[:, :r].copy() for v in V]
    for f in init:
        f[:, 1] = f[:, 0] * (1.0 + 1e-7)
    S = specs_for(qs)
    cfg = cp.ALSApproxConfig(max_sweeps=4, stall=-np.inf, reg=1e-10)
    als_variant(9, 0)
    assert cp.als_plan(qs, R, r)["kernel"] == "als_w"
    tw = []
    a = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init), trace=tw)
    als_variant(8, 0)
    tr = []
    b = cp.cp_approx_als(cp.CPTensor(S, V), r, cfg, init=cp.CPTensor(S, init), trace=tr)
    assert torch.equal(a.data, b.data) and tw == tr
    assert np.all(np.isfinite(a.data.cpu().numpy()))
    # an all-zero target (zero pivots) takes the same route: zeros, not an error (cp.py:176-177)
    als_variant(9, 0)
    Z = cp.CPTensor(S, [np.zeros((q, R)) for q in qs])
    z = cp.cp_approx_als(Z, r, cfg, init=cp.CPTensor(S, init))
    assert torch.count_nonzero(z.data).item() == 0


@pytest.mark.parametrize("variant,cluster", [(0, 0), (1, 0), (8, 0)])
def test_als_near_singular_gram_trace_rule(als_variant, variant, cluster):
    """Near-singular normal equations under the reference trace rule (cp.py:171-173:
    lambda = 1e-12 tr(A)/r): two init columns equal up to 1e-13 make every Gram product
    numerically rank deficient (cond ~1e12).  np.linalg.solve succeeds there (no lstsq
    fallback), so the fit must exist, stay finite and agree with the oracle within the
    problem's own sensitivity (the oracle against itself on a 1e-13-perturbed init)."""
    als_variant(variant, cluster)
    rng = np.random.default_rng(31)
    qs, R, r = (40, 36, 48, 40), 64, 6
    V = rand_factors(rng, qs, R, 0.3)
    init = [v[:, :r].copy() for v in V]
    for f in init:
        f[:, 1] = f[:, 0] * (1.0 + 1e-13)
    out, ref, trace, otrace = _als_case(V, init, 5, None)
    assert np.all(np.isfinite(out.data.cpu().numpy()))
    # the problem's own sensitivity: the oracle on a 1e-13-perturbed init
    init_p = [f * (1.0 + 1e-13 * np.random.default_rng(5).standard_normal(f.shape)) for f in init]
    ptrace = []
    pref = ocp.als(V, init_p, 5, lam=None, trace=ptrace)
    sens_t = float(np.max(np.abs(np.array(ptrace) - np.array(otrace)) / np.array(otrace)))
    sens_f = metrics.cp_rel_diff(ref, pref)
    assert sens_t > 1e-7   # (really ill-conditioned: the reference's own rounding moves the fit)
    assert float(np.max(np.abs(np.array(trace) - np.array(otrace)) / np.array(otrace))) <= 10 * sens_t
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= 10 * sens_f


@pytest.mark.parametrize("d", [10, 16])
def test_many_modes(d):
    """More modes than the fused kernels hold (d > 8): ALS through the streamed variant,
    inner product and operator apply up to 16 modes, against the oracle."""
    from oracle import operators as oops
    rng = np.random.default_rng(d)
    qs = tuple(int(q) for q in rng.integers(5, 9, size=d))
    R, r = 14, 3
    V = rand_factors(rng, qs, R, 0.6)
    init = [v[:, :r].copy() for v in V]
    assert cp.als_plan(qs, R, r)["kernel"] == "als_generic"
    out, ref, trace, otrace = _als_case(V, init, 4, 1e-10)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= TOL_TRUNC
    S = specs_for(qs)
    T = cp.CPTensor(S, V)
    assert abs(cp.inner_product(T, T) - ocp.inner_product(V, V).real) <= 1e-12 * abs(cp.inner_product(T, T))
    mats = [[rng.standard_normal((q, q)) / q if k == t else None for k, q in enumerate(qs)] for t in range(3)]
    L = operators.SeparableOperator(S, (0.5, -1.0, 2.0), tuple(tuple(m) for m in mats))
    got = operators.apply(L, T).to_numpy()
    exp = oops.apply([0.5, -1.0, 2.0], mats, V)
    assert metrics.cp_rel_diff(exp, got) <= 1e-13
