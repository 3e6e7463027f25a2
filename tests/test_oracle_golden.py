"""Pin the CPU oracle against golden vectors produced by the real reference package
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import load_golden, unpack_cp, unpack_ht
from oracle import cp_als, explicit, ht_hsvd, implicit, metrics, operators


@pytest.fixture(scope="module")
def g_cp():
    return load_golden("cp_als")


def test_cp_als_matches_reference_golden(g_cp):
    for name in g_cp["names"]:
        name = str(name)
        V = unpack_cp(g_cp, f"{name}_V")
        init = unpack_cp(g_cp, f"{name}_init")
        ref = unpack_cp(g_cp, f"{name}_out")
        sweeps, lam, stall, r = g_cp[f"{name}_meta"]
        trace = []
        out = cp_als.als(V, init, int(sweeps), lam=None if lam < 0 else lam, stall=stall, trace=trace)
        assert len(trace) == len(g_cp[f"{name}_trace"]), name
        np.testing.assert_allclose(trace, g_cp[f"{name}_trace"], rtol=1e-6, atol=1e-9)
        rel = metrics.cp_rel_diff(ref, out)
        assert rel < 1e-12, (name, rel)


def test_cp_als_complex_reference_arithmetic(g_cp):
    V = unpack_cp(g_cp, "complex_V")
    init = unpack_cp(g_cp, "complex_init")
    ref = unpack_cp(g_cp, "complex_out")
    trace = []
    out = cp_als.als(V, init, 40, lam=None, stall=1e-13, trace=trace)
    assert len(trace) == len(g_cp["complex_trace"])
    # same numpy operations in the same order as the reference: bitwise identical
    for a, b in zip(out, ref):
        assert np.array_equal(a, b)


def test_inner_product_and_metric_golden(g_cp):
    f = unpack_cp(g_cp, "ip_f")
    g = unpack_cp(g_cp, "ip_g")
    assert abs(cp_als.inner_product(f, g) - complex(g_cp["ip_fg"])) < 1e-12 * abs(complex(g_cp["ip_fg"])) + 1e-14
    assert abs(cp_als.norm(f) - float(g_cp["ip_norm_f"])) < 1e-13 * float(g_cp["ip_norm_f"])
    f2 = [x * (1 + 1e-9) for x in f]
    rel = metrics.cp_rel_diff(f, f2)
    assert abs(rel - float(g_cp["metric_rel"])) < 1e-15
    assert abs(rel - ((1 + 1e-9) ** 3 - 1)) < 1e-13  # resolves a 3e-9 perturbation (3 modes)


def test_ht_truncate_matches_reference_golden():
    g = load_golden("ht")
    for name in g["names"]:
        name = str(name)
        d, q, rin, rmax, eps, est = g[f"{name}_meta"]
        nodes = ht_hsvd.balanced_tree(int(d))
        fin, tin = unpack_ht(g, f"{name}_in", nodes)
        fout, tout = unpack_ht(g, f"{name}_out", nodes)
        h = (nodes, fin, tin)
        red, my_est = ht_hsvd.truncate(h, int(rmax), float(eps))
        assert abs(my_est - est) <= 1e-9 * max(1.0, float(g[f"{name}_norm_in"])), name
        ref = (nodes, fout, tout)
        # compare represented tensors (eigenvector gauge differs), stable metric
        rel = metrics.ht_rel_diff(ref, red)
        assert rel < 1e-12, (name, rel)
        assert abs(ht_hsvd.norm(h) - float(g[f"{name}_norm_in"])) < 1e-12 * float(g[f"{name}_norm_in"])


def test_operator_apply_golden():
    g = load_golden("operators")
    f = unpack_cp(g, "gal_f")
    nterms = int(g["gal_nterms"])
    mats = [[g.get(f"gal_E{t}_{k}") for k in range(len(f))] for t in range(nterms)]
    out = operators.apply(list(g["gal_weights"]), mats, f)
    for a, b in zip(out, unpack_cp(g, "gal_out")):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-14)
    fr = unpack_cp(g, "col_f")
    D, a = g["col_D"], g["col_a"]
    mats = [[D if k == t else None for k in range(3)] for t in range(3)]
    out = operators.apply(list(-a), mats, fr)
    for x, y in zip(out, unpack_cp(g, "col_out")):
        np.testing.assert_allclose(x, y, rtol=0, atol=1e-14)


def test_explicit_fused_trajectory_golden():
    g = load_golden("explicit")
    q, d, r, dt, steps, sweeps, lam = g["meta"]
    d, r, steps, sweeps = int(d), int(r), int(steps), int(sweeps)
    D, a = g["D"], g["a"]
    mats = [[D if k == t else None for k in range(d)] for t in range(d)]
    f0 = unpack_cp(g, "step0")
    got = {}
    explicit.run_fused(f0, list(-a), mats, dt, r, steps, sweeps, lam,
                       callback=lambda n, f: got.__setitem__(n, f))
    for n in range(1, steps + 1):
        rel = metrics.cp_rel_diff(unpack_cp(g, f"step{n}"), got[n])
        assert rel < 1e-12, (n, rel)


def test_implicit_step_golden():
    g = load_golden("implicit")
    q, d, r, dt, sweeps, lam = g["meta"]
    d, sweeps = int(d), int(sweeps)
    D, a = g["D"], g["a"]
    mats = [[None] * d] + [[D if k == i else None for k in range(d)] for i in range(d)]
    eta = [1.0] + list(dt * a)
    zeta = [1.0] + [0.0] * d
    tables = implicit.build_tables(mats, eta, zeta, [int(q)] * d)
    f0 = unpack_cp(g, "f0")
    np.testing.assert_allclose(implicit.build_M(1, f0, tables), g["M1"].real, atol=1e-12)
    np.testing.assert_allclose(implicit.build_gamma(1, f0, f0, tables, "reference"),
                               g["gamma1_reference"].real, atol=1e-12)
    for orient, key in (("reference", "out_reference_orientation"), ("corrected", "out_corrected")):
        out, done, _ = implicit.step(f0, tables, sweeps, lam, orientation=orient)
        assert done == sweeps
        rel = metrics.cp_rel_diff(unpack_cp(g, key), out)
        assert rel < 1e-12, (orient, rel)


def _complex_ex_setup():
    g = load_golden("complex")
    nt = int(g["ex_nterms"])
    mats = [[g[f"ex_E{t}_{k}"] if f"ex_E{t}_{k}" in g else None for k in range(2)] for t in range(nt)]
    return g, list(g["ex_weights"]), mats


def test_complex_rank_reduce_and_split_recipe_golden():
    """Oracle vs the reference run natively in complex128 (rank_reduce_als with its
    complex random terms; the explicit split recipe on the Galerkin basis)."""
    from oracle import cp_als as ocp
    from oracle import explicit as oex
    g, w, mats = _complex_ex_setup()
    out = ocp.rank_reduce(unpack_cp(g, "rr_f"), 3, 1e-9)
    assert metrics.cp_rel_diff(unpack_cp(g, "rr_out"), out) <= 1e-12
    red = lambda t, init: ocp.rank_reduce(t, 3, 1e-8)  # noqa: E731
    f0 = unpack_cp(g, "ex_step0")
    traj = [f0, oex.startup_split(f0, w, mats, 1e-2, 3, red)]
    for _ in range(2):
        traj.append(oex.ab2_split(traj[-2], traj[-1], w, mats, 1e-2, 3, red))
    for n, f in enumerate(traj):
        assert metrics.cp_rel_diff(unpack_cp(g, f"ex_step{n}"), f) <= 1e-10, n


def test_implicit_forced_step_golden():
    """Forced steps (implicit.py:140-152) of the real reference: Gauss-Seidel with fixed
    sweeps and the default Jacobi schedule (delta_beta = 4) stopping on eps_tol, both
    orientations; the oracle reproduces the sweep counts and the states."""
    g = load_golden("implicit_forced")
    q, d, r, dt, lam = g["meta"]
    d = int(d)
    D, a = g["D"], g["a"]
    mats = [[None] * d] + [[D if k == i else None for k in range(d)] for i in range(d)]
    tables = implicit.build_tables(mats, [1.0] + list(dt * a), [1.0] + [0.0] * d, [int(q)] * d)
    f0, force = unpack_cp(g, "f0"), unpack_cp(g, "forcing")
    for case in ("gs", "jac"):
        eps_tol, max_sweeps, delta_beta, jac = g[f"{case}_cfg"]
        for i, (orient, key) in enumerate((("reference", "out_reference_orientation"), ("corrected", "out_corrected"))):
            out, done, _ = implicit.step(f0, tables, int(max_sweeps), lam, "jacobi" if jac else "gauss-seidel",
                                         float(delta_beta), float(eps_tol), orient, forcing=force, dt=float(dt))
            assert done == int(g[f"{case}_sweeps"][i]), (case, orient, done)
            rel = metrics.cp_rel_diff(unpack_cp(g, f"{case}_{key}"), out)
            assert rel < 1e-11, (case, orient, rel)


def test_ht_truncate_nonbalanced_trees_golden():
    """Reference hSVD on caterpillar and uneven dimension trees (ht.py:55-76, 313-372)."""
    from conftest import tree_nodes, unpack_ht
    g = load_golden("ht_trees")
    for name in g["names"]:
        name = str(name)
        nodes = tree_nodes(g, name)
        d, q, rin, rmax, eps, est = g[f"{name}_meta"]
        fin, tin = unpack_ht(g, f"{name}_in", nodes)
        fout, tout = unpack_ht(g, f"{name}_out", nodes)
        red, oest = ht_hsvd.truncate((nodes, fin, tin), int(rmax), float(eps))
        assert abs(oest - est) <= 1e-10 * max(1.0, float(g[f"{name}_norm_in"])), (name, oest, est)
        assert metrics.ht_rel_diff((nodes, fout, tout), red) <= 1e-10, name
