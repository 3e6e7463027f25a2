"""Generate golden fixtures by running the REAL reference ``tensorpde`` package.

Run in the build container (where ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports ``/root/reference/pkg/src/tensorpde`` read-only, applies the shims
of SURVEY.md 8(c) (S1 even-Q spec bypass, S2 fixed lambda, S3 fixed sweep
count, S4 dense-matrix apply, S5-S8 implicit tables / direct solve /
orientation / schedule), and writes small seeded input/output vectors to
``tests/golden/*.npz``.  The tests pin ``oracle/`` against these files; the
GPU box never reads ``/root/reference``.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from tensorpde import cp, ht, implicit, operators  # noqa: E402
from tensorpde.basis import BasisSpec, FactorKind, factor_matrix  # noqa: E402
from tensorpde.models import spiral_matrix  # noqa: E402


def spec(q, b=np.pi):
    """S1: build a BasisSpec without the odd-Q validation (frozen dataclass bypass)."""
    s = object.__new__(BasisSpec)
    object.__setattr__(s, "Q", int(q))
    object.__setattr__(s, "b", float(b))
    return s


def fixed_lambda(lam):
    """S2: replace the trace-scaled regulariser with a fixed lambda (LU solve kept)."""
    def solve(gram, rhs):
        return np.linalg.solve(gram + lam * np.eye(gram.shape[0]), rhs)
    return solve


def real_cp(specs, r, rng, scale=1.0):
    return cp.CPTensor(specs, [scale * rng.standard_normal((s.Q, r)) for s in specs])


def fourier_diff_matrix(q):
    """Even-Q Fourier collocation derivative on [0, 2pi) (same as the product's builder)."""
    h = 2 * np.pi / q
    D = np.zeros((q, q))
    for i in range(q):
        for j in range(q):
            if i != j:
                D[i, j] = 0.5 * (-1) ** (i - j) / np.tan((i - j) * h / 2)
    return D


def dense_apply(weights, mats, f):
    """S4: operators.apply (operators.py:48-62) with dense factor matrices."""
    blocks = [[] for _ in f.specs]
    for w, row in zip(weights, mats):
        for k in range(f.ndim):
            col = f.factors[k].copy() if row[k] is None else row[k] @ f.factors[k]
            if k == 0:
                col = col * w
            blocks[k].append(col)
    return cp.CPTensor(f.specs, [np.hstack(c) for c in blocks])


def pack_cp(prefix, f, store):
    for k, m in enumerate(f.factors):
        store[f"{prefix}_{k}"] = m
    store[f"{prefix}_d"] = np.array(len(f.factors))


def gen_cp_als():
    store = {}
    orig = cp._solve_gram
    cases = [
        # name, Qs, R, r, sweeps, lam (None = reference trace rule), stall, seed
        ("small_fixed", (5, 7, 3), 6, 2, 15, 1e-10, -np.inf, 1),
        ("cfg1_shape", (16,) * 6, 40, 8, 20, 1e-10, -np.inf, 2),
        ("ref_rule_stall", (9, 8, 7, 6), 10, 3, 60, None, 1e-13, 3),
        ("rank1", (12, 12, 12), 5, 1, 10, 1e-10, -np.inf, 4),
        ("r32_q64", (64,) * 4, 96, 32, 6, 1e-10, -np.inf, 5),
    ]
    names = []
    for name, qs, R, r, sweeps, lam, stall, seed in cases:
        rng = np.random.default_rng(seed)
        specs = tuple(spec(q) for q in qs)
        V = real_cp(specs, R, rng, scale=1.0 / np.sqrt(qs[0]))
        init = cp.CPTensor(specs, [fk[:, :r].copy() for fk in V.factors])
        cp._solve_gram = fixed_lambda(lam) if lam is not None else orig
        trace = []
        out = cp.cp_approx_als(V, r, cp.ALSApproxConfig(max_sweeps=sweeps, tol=0.0, stall=stall),
                               init=init, trace=trace)
        cp._solve_gram = orig
        pack_cp(f"{name}_V", V, store)
        pack_cp(f"{name}_init", init, store)
        pack_cp(f"{name}_out", out, store)
        store[f"{name}_trace"] = np.array(trace)
        store[f"{name}_meta"] = np.array([sweeps, -1.0 if lam is None else lam, stall, r], dtype=float)
        names.append(name)
    # a complex-valued case in the reference's native arithmetic (trace rule, default stall)
    rng = np.random.default_rng(6)
    specs = tuple(spec(q) for q in (5, 7, 3))
    Vc = cp.random_cp(specs, 4, rng)
    initc = cp.random_cp(specs, 2, rng)
    trace = []
    outc = cp.cp_approx_als(Vc, 2, cp.ALSApproxConfig(max_sweeps=40), init=initc, trace=trace)
    pack_cp("complex_V", Vc, store)
    pack_cp("complex_init", initc, store)
    pack_cp("complex_out", outc, store)
    store["complex_trace"] = np.array(trace)
    store["names"] = np.array(names)
    # inner products
    f = real_cp(tuple(spec(q) for q in (6, 5, 4)), 3, rng)
    g = real_cp(tuple(spec(q) for q in (6, 5, 4)), 4, rng)
    pack_cp("ip_f", f, store)
    pack_cp("ip_g", g, store)
    store["ip_fg"] = np.array(cp.inner_product(f, g))
    store["ip_norm_f"] = np.array(cp.norm(f))
    # stable difference metric computed with reference primitives only
    h = cp.add(f, cp.scale(cp.CPTensor(f.specs, [x * (1 + 1e-9) for x in f.factors]), -1.0))
    store["metric_rel"] = np.array(ht.norm(ht.from_cp(h)) / cp.norm(f))
    np.savez_compressed(OUT / "cp_als.npz", **store)


def pack_ht(prefix, h, store):
    for i, u in enumerate(h.frames):
        if u is not None:
            store[f"{prefix}_F{i}"] = u
    for i, b in enumerate(h.transfers):
        if b is not None:
            store[f"{prefix}_B{i}"] = b


def gen_ht():
    store = {}
    cases = [
        # name, d, Q, rank_in, r_max, eps, seed, random transfers?
        ("inflated", 4, 6, 2, 2, 0.0, 11, False),
        ("d8_random", 8, 10, 6, 3, 0.0, 12, True),
        ("d5_eps", 5, 7, 4, 4, 1e-3, 13, True),
        ("d3_cap", 3, 9, 5, 2, 0.0, 14, True),
        ("d2", 2, 8, 4, 2, 0.0, 15, True),
    ]
    names = []
    for name, d, q, rin, rmax, eps, seed, rand in cases:
        rng = np.random.default_rng(seed)
        specs = tuple(spec(q) for _ in range(d))
        tree = ht.balanced_tree(d)
        if rand:
            frames = [None] * len(tree.nodes)
            transfers = [None] * len(tree.nodes)
            for i, node in enumerate(tree.nodes):
                if node.is_leaf:
                    frames[i] = rng.standard_normal((q, rin))
                else:
                    transfers[i] = rng.standard_normal((rin, rin, 1 if i == 0 else rin))
            h = ht.HTTensor(specs, tree, frames, transfers)
        else:
            f = real_cp(specs, rin, rng)
            h0 = ht.from_cp(f)
            h = ht.add(h0, h0)
        red, est = ht.truncate(h, rmax, eps)
        pack_ht(f"{name}_in", h, store)
        pack_ht(f"{name}_out", red, store)
        store[f"{name}_meta"] = np.array([d, q, rin, rmax, eps, est])
        store[f"{name}_norm_in"] = np.array(ht.norm(h))
        names.append(name)
    store["names"] = np.array(names)
    np.savez_compressed(OUT / "ht.npz", **store)


def _tree(ndim, split):
    """DimensionTree built in preorder with a custom split rule (ht.py:55-76 accepts any)."""
    nodes = []

    def build(dims, parent):
        idx = len(nodes)
        nodes.append(None)
        if len(dims) == 1:
            nodes[idx] = ht.TreeNode(dims, parent, -1, -1)
        else:
            cut = split(len(dims))
            left = build(dims[:cut], idx)
            right = build(dims[cut:], idx)
            nodes[idx] = ht.TreeNode(dims, parent, left, right)
        return idx

    build(tuple(range(ndim)), -1)
    return ht.DimensionTree(tuple(nodes))


def gen_ht_trees():
    """hSVD truncation (ht.py:313-372) of the reference on NON-balanced dimension trees:
    left and right caterpillars and a 1/3-2/3 split, random frames/transfers."""
    store = {}
    cases = [("cat_left", 5, 7, 4, 2, 0.0, 31, lambda n: n - 1),
             ("cat_right", 6, 6, 5, 3, 0.0, 32, lambda n: 1),
             ("third", 7, 8, 5, 3, 1e-3, 33, lambda n: max(1, n // 3))]
    names = []
    for name, d, q, rin, rmax, eps, seed, split in cases:
        rng = np.random.default_rng(seed)
        specs = tuple(spec(q) for _ in range(d))
        tree = _tree(d, split)
        frames = [None] * len(tree.nodes)
        transfers = [None] * len(tree.nodes)
        for i, node in enumerate(tree.nodes):
            if node.is_leaf:
                frames[i] = rng.standard_normal((q, rin))
            else:
                transfers[i] = rng.standard_normal((rin, rin, 1 if i == 0 else rin))
        h = ht.HTTensor(specs, tree, frames, transfers)
        red, est = ht.truncate(h, rmax, eps)
        pack_ht(f"{name}_in", h, store)
        pack_ht(f"{name}_out", red, store)
        store[f"{name}_tree"] = np.array([[n.parent, n.left, n.right] for n in tree.nodes])
        store[f"{name}_dims"] = np.array([n.dims[0] if n.is_leaf else -1 for n in tree.nodes])
        store[f"{name}_meta"] = np.array([d, q, rin, rmax, eps, est])
        store[f"{name}_norm_in"] = np.array(ht.norm(h))
        names.append(name)
    store["names"] = np.array(names)
    np.savez_compressed(OUT / "ht_trees.npz", **store)


def gen_operators():
    store = {}
    rng = np.random.default_rng(21)
    specs = (BasisSpec(5, 1.5), BasisSpec(7, 2.0), BasisSpec(3, 0.8))
    op = operators.advection_operator(spiral_matrix(3, 2.0), specs)
    f = cp.random_cp(specs, 2, rng)
    g = operators.apply(op, f)
    pack_cp("gal_f", f, store)
    pack_cp("gal_out", g, store)
    store["gal_weights"] = np.array(op.weights)
    for t, row in enumerate(op.factors):
        for k, kind in enumerate(row):
            if kind is not FactorKind.IDENTITY:
                store[f"gal_E{t}_{k}"] = factor_matrix(specs[k], kind)
    store["gal_nterms"] = np.array(op.n_terms)
    # real collocation advection operator (BASELINE cfg0 form), via the S4 shim
    qs = 8
    specs6 = tuple(spec(qs) for _ in range(3))
    D = fourier_diff_matrix(qs)
    a = np.array([1.0, 0.5, -0.75])
    mats = [[D if k == t else None for k in range(3)] for t in range(3)]
    fr = real_cp(specs6, 3, rng)
    gr = dense_apply(-a, mats, fr)
    pack_cp("col_f", fr, store)
    pack_cp("col_out", gr, store)
    store["col_D"] = D
    store["col_a"] = a
    np.savez_compressed(OUT / "operators.npz", **store)


def gen_explicit():
    """Fused AB2/RK2 trajectory composed from reference primitives (cp.add/scale,
    S4 dense apply, cp_approx_als with S2/S3)."""
    store = {}
    rng = np.random.default_rng(31)
    q, d, r, dt, steps, sweeps, lam = 8, 3, 3, 1e-2, 6, 10, 1e-10
    specs = tuple(spec(q) for _ in range(d))
    D = fourier_diff_matrix(q)
    a = np.array([1.0, 0.5, -0.75])
    mats = [[D if k == t else None for k in range(d)] for t in range(d)]
    x = 2 * np.pi * np.arange(q) / q
    facs = []
    for k in range(d):
        cols = [np.exp(np.sin(x + rng.uniform(0, 2 * np.pi))) for _ in range(2)]
        facs.append(np.stack(cols, axis=1))
    facs[0] = facs[0] * rng.uniform(0.5, 1.5, size=2)
    f0 = cp.CPTensor(specs, facs)
    f0 = cp.add(f0, cp.CPTensor(specs, [1e-8 * rng.standard_normal((q, r - 2)) for _ in range(d)]))
    orig = cp._solve_gram
    cp._solve_gram = fixed_lambda(lam)
    cfg = cp.ALSApproxConfig(max_sweeps=sweeps, tol=0.0, stall=-np.inf)

    def red(t, init):
        if t.rank <= r:
            return t
        return cp.cp_approx_als(t, r, cfg, init=init)

    L = lambda f: dense_apply(-a, mats, f)  # noqa: E731
    half = red(cp.add(f0, cp.scale(L(f0), 0.5 * dt)), f0)
    f1 = red(cp.add(f0, cp.scale(L(half), dt)), f0)
    traj = [f0, f1]
    for _ in range(2, steps + 1):
        prev, cur = traj[-2], traj[-1]
        w = cp.add(cp.scale(cur, 3.0), cp.scale(prev, -1.0))
        traj.append(red(cp.add(cur, cp.scale(L(w), 0.5 * dt)), cur))
    cp._solve_gram = orig
    for n, f in enumerate(traj):
        pack_cp(f"step{n}", f, store)
    store["meta"] = np.array([q, d, r, dt, steps, sweeps, lam])
    store["D"] = D
    store["a"] = a
    np.savez_compressed(OUT / "explicit.npz", **store)


def gen_implicit():
    """One implicit-Euler step through the reference ``implicit.step`` with S5-S8."""
    store = {}
    rng = np.random.default_rng(41)
    q, d, r, dt, sweeps, lam = 6, 3, 2, 5e-2, 4, 1e-10
    specs = tuple(spec(q) for _ in range(d))
    D = fourier_diff_matrix(q)
    a = np.array([1.0, 0.5, -0.75])
    # A = I + dt sum a_i D_i  (terms: identity, then D on mode i), B = I
    mats = [[None] * d] + [[D if k == i else None for k in range(d)] for i in range(d)]
    eta = (1.0,) + tuple(dt * a)
    zeta = (1.0,) + (0.0,) * d
    ra = len(eta)
    pairs, source = [], []
    for k in range(d):
        full = [np.eye(q) if mats[e][k] is None else mats[e][k] for e in range(ra)]
        pairs.append(np.array([[full[e].T @ full[z] for z in range(ra)] for e in range(ra)], dtype=complex))
        source.append(np.array([full[e].T for e in range(ra)], dtype=complex))
    eta_c = np.asarray(eta, dtype=complex)
    zeta_c = np.asarray(zeta, dtype=complex)
    L = operators.SeparableOperator(specs, tuple(-a), tuple(tuple(FactorKind.DERIVATIVE if k == i else FactorKind.IDENTITY
                                                                   for k in range(d)) for i in range(d)))
    pair = operators.CrankNicolsonPair(specs, dt, eta, zeta, tuple(tuple(FactorKind.IDENTITY for _ in range(d))
                                                                   for _ in range(ra)), L)
    tables = implicit.OperatorTables(pair, pairs, source, np.outer(eta_c, eta_c), np.outer(eta_c, zeta_c))
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=1.0,
                                 schedule="gauss-seidel")
    ws = object.__new__(implicit.StepWorkspace)
    ws.pair, ws.config, ws.tables, ws._pool = pair, cfg, tables, None
    f0 = real_cp(specs, r, rng)
    orig_solve, orig_gamma = implicit.solve_beta, implicit.build_gamma

    def direct(M, gamma, beta_init, config):                     # S6
        return np.linalg.solve(M + lam * np.eye(M.shape[0]), gamma), 0, 0.0

    def gamma_fixed(qq, beta_new, beta_old, tab, forcing=None):  # S7
        had = implicit._term_grams(tab, beta_new, beta_old, qq)
        gam = np.einsum("ez,ezij,ezac,cj->ia", tab.KR, had, tab.pairs[qq], beta_old[qq], optimize=True)
        return gam.reshape(-1)

    implicit.solve_beta = direct
    out_ref = implicit.step(f0, pair, None, cfg, workspace=ws)
    implicit.build_gamma = gamma_fixed
    out_fix = implicit.step(f0, pair, None, cfg, workspace=ws)
    implicit.solve_beta, implicit.build_gamma = orig_solve, orig_gamma
    pack_cp("f0", f0, store)
    pack_cp("out_reference_orientation", out_ref, store)
    pack_cp("out_corrected", out_fix, store)
    store["meta"] = np.array([q, d, r, dt, sweeps, lam])
    store["D"] = D
    store["a"] = a
    # M and gamma blocks for mode 1 at the initial iterate (reference builders)
    beta = [fk.astype(complex) for fk in f0.factors]
    store["M1"] = implicit.build_M(1, beta, tables)
    store["gamma1_reference"] = orig_gamma(1, beta, beta, tables)
    np.savez_compressed(OUT / "implicit.npz", **store)


def gen_implicit_forced():
    """Forced implicit steps through the reference ``implicit.step`` (forcing block
    implicit.py:140-152) with S5/S6: Gauss-Seidel (4 fixed sweeps) and the reference
    default Jacobi schedule (delta_beta = 4, eps_tol = 1e-4 -> the convergence stop),
    each in the reference orientation (native build_gamma) and the corrected one
    (S7 for the b_old block; the forcing block is the reference's own, taken as
    build_gamma(forcing) - build_gamma(None))."""
    store = {}
    rng = np.random.default_rng(43)
    q, d, r, rf, dt, lam = 6, 3, 2, 2, 5e-2, 1e-10
    specs = tuple(spec(q) for _ in range(d))
    D = fourier_diff_matrix(q)
    a = np.array([1.0, 0.5, -0.75])
    mats = [[None] * d] + [[D if k == i else None for k in range(d)] for i in range(d)]
    eta = (1.0,) + tuple(dt * a)
    zeta = (1.0,) + (0.0,) * d
    ra = len(eta)
    pairs, source = [], []
    for k in range(d):
        full = [np.eye(q) if mats[e][k] is None else mats[e][k] for e in range(ra)]
        pairs.append(np.array([[full[e].T @ full[z] for z in range(ra)] for e in range(ra)], dtype=complex))
        source.append(np.array([full[e].T for e in range(ra)], dtype=complex))
    eta_c = np.asarray(eta, dtype=complex)
    zeta_c = np.asarray(zeta, dtype=complex)
    L = operators.SeparableOperator(specs, tuple(-a), tuple(tuple(FactorKind.DERIVATIVE if k == i else FactorKind.IDENTITY
                                                                   for k in range(d)) for i in range(d)))
    pair = operators.CrankNicolsonPair(specs, dt, eta, zeta, tuple(tuple(FactorKind.IDENTITY for _ in range(d))
                                                                   for _ in range(ra)), L)
    tables = implicit.OperatorTables(pair, pairs, source, np.outer(eta_c, eta_c), np.outer(eta_c, zeta_c))
    f0 = real_cp(specs, r, rng)
    forcing = real_cp(specs, rf, rng, 0.5)
    orig_solve, orig_gamma = implicit.solve_beta, implicit.build_gamma

    def direct(M, gamma, beta_init, config):                     # S6
        return np.linalg.solve(M + lam * np.eye(M.shape[0]), gamma), 0, 0.0

    def gamma_fixed(qq, beta_new, beta_old, tab, forcing=None):  # S7 + the reference forcing block
        had = implicit._term_grams(tab, beta_new, beta_old, qq)
        gam = np.einsum("ez,ezij,ezac,cj->ia", tab.KR, had, tab.pairs[qq], beta_old[qq], optimize=True).reshape(-1)
        if forcing is not None:
            gam = gam + (orig_gamma(qq, beta_new, beta_old, tab, forcing) - orig_gamma(qq, beta_new, beta_old, tab))
        return gam

    cases = {"gs": dict(eps_tol=0.0, max_sweeps=4, delta_beta=1.0, schedule="gauss-seidel"),
             "jac": dict(eps_tol=1e-4, max_sweeps=60, delta_beta=4.0, schedule="jacobi")}
    implicit.solve_beta = direct
    try:
        for name, kw in cases.items():
            cfg = implicit.ALSStepConfig(dt=dt, **kw)
            ws = object.__new__(implicit.StepWorkspace)
            ws.pair, ws.config, ws.tables, ws._pool = pair, cfg, tables, None
            log_r, log_c = {}, {}
            implicit.build_gamma = orig_gamma
            out_ref = implicit.step(f0, pair, forcing, cfg, workspace=ws, log=log_r)
            implicit.build_gamma = gamma_fixed
            out_fix = implicit.step(f0, pair, forcing, cfg, workspace=ws, log=log_c)
            pack_cp(f"{name}_out_reference_orientation", out_ref, store)
            pack_cp(f"{name}_out_corrected", out_fix, store)
            store[f"{name}_sweeps"] = np.array([log_r["sweeps"], log_c["sweeps"]])
            store[f"{name}_cfg"] = np.array([kw["eps_tol"], kw["max_sweeps"], kw["delta_beta"],
                                             1.0 if kw["schedule"] == "jacobi" else 0.0])
    finally:
        implicit.solve_beta, implicit.build_gamma = orig_solve, orig_gamma
    pack_cp("f0", f0, store)
    pack_cp("forcing", forcing, store)
    store["meta"] = np.array([q, d, r, dt, lam])
    store["D"] = D
    store["a"] = a
    np.savez_compressed(OUT / "implicit_forced.npz", **store)


def gen_io():
    """Reference-written tensor files (io.save_tensor, io.py:55-71) + their decoded arrays."""
    from tensorpde import io as rio
    rng = np.random.default_rng(17)
    specs = (BasisSpec(5, 1.5), BasisSpec(7, 2.0), BasisSpec(3, 1.0))
    f = real_cp(specs, 3, rng)
    rio.save_tensor(OUT / "io_cp.tensor", f)
    store = {}
    pack_cp("cp", f, store)
    specs4 = (BasisSpec(5, 1.5), BasisSpec(3, 2.0), BasisSpec(7, 1.0), BasisSpec(5, 2.5))
    h = ht.from_cp(real_cp(specs4, 2, rng))
    h, _ = ht.truncate(ht.add(h, h), r_max=3, eps=1e-14)     # node ranks vary (reference test_io.py:46-50)
    rio.save_tensor(OUT / "io_ht.tensor", h)
    pack_ht("ht", h, store)
    np.savez_compressed(OUT / "io.npz", **store)


def gen_diagnostics():
    """Reference diagnostics on fixed inputs (diagnostics.py:31-143)."""
    from tensorpde import diagnostics as rdiag
    from tensorpde import models
    from tensorpde.basis import integration_weights
    store = {}
    rng = np.random.default_rng(23)
    x, y = rng.standard_normal(50), rng.standard_normal(50)
    store["nmae_x"], store["nmae_y"], store["nmae"] = x, y, rdiag.nmae(x, y)
    t = np.linspace(0.0, 4.0, 30)
    series = 3.0 * np.exp(-1.7 * t) + 1e-6
    store["fit_t"], store["fit_series"] = t, series
    store["fit_rate"] = rdiag.fit_decay_rate(t, series)
    store["fit_rate_floor"] = rdiag.fit_decay_rate(t, series, floor=1e-6)
    spec = models.BGKSpec(Q=11)
    f = models.maxwellian_cp(spec)
    rep = rdiag.moments(f, spec)
    pack_cp("mw", f, store)
    for p in (0, 1, 2):
        store[f"mw_w{p}"] = np.stack([integration_weights(s, p) for s in f.specs])
    store["mw_R"] = spec.R
    store["mw_out"] = np.concatenate([[rep.mean_density], rep.mean_velocity, [rep.mean_temperature]])
    np.savez_compressed(OUT / "diagnostics.npz", **store)


def gen_complex():
    """Complex128 path in the reference's native arithmetic, no shims:
    rank_reduce_als with its complex random terms (cp.py:337-366) and the reference's
    explicit split recipe (explicit.py:85-103) on the Fourier Galerkin basis with the
    reference advection operator (operators.py:65-87)."""
    from tensorpde import explicit
    store = {}
    rng = np.random.default_rng(41)
    specs = (BasisSpec(5, 1.5), BasisSpec(7, 2.0), BasisSpec(3, 0.8))
    # exactly rank 2: the adaptive loop (ranks 1, 2) stops at rank 2 with a converged
    # fit (a non-converged or noise-fitting best rank would make the stall-terminated
    # result sensitive at the 1e-8 level)
    f = cp.random_cp(specs, 2, rng)
    red = cp.rank_reduce_als(f, 3, 1e-9)
    pack_cp("rr_f", f, store)
    pack_cp("rr_out", red, store)
    # a REAL target (exactly rank 2): the reference still draws complex random terms, so its
    # fit is complex -- pins rank_reduce_als(..., draws="reference") on real data
    fr = cp.CPTensor(specs, [np.random.default_rng(43).standard_normal((s.Q, 2)) for s in specs])
    redr = cp.rank_reduce_als(fr, 3, 1e-9)
    pack_cp("rrr_f", fr, store)
    pack_cp("rrr_out", redr, store)
    # explicit split recipe: 2-D sheared advection, Galerkin Q = 9
    specs2 = (BasisSpec(9, 3.0), BasisSpec(9, 3.0))
    op = operators.advection_operator(spiral_matrix(2, 2.0), specs2)
    f0 = cp.scale(cp.random_cp(specs2, 2, rng), 0.5)
    cfg = explicit.ExplicitConfig(dt=1e-2, r_max=3, eps_rank=1e-8)
    traj = [f0, explicit.startup_step(f0, op, cfg)]
    for _ in range(2):
        traj.append(explicit.ab2_step(traj[-2], traj[-1], op, cfg))
    for n, g in enumerate(traj):
        pack_cp(f"ex_step{n}", g, store)
    store["ex_weights"] = np.array(op.weights)
    for t, row in enumerate(op.factors):
        for k, kind in enumerate(row):
            if kind is not FactorKind.IDENTITY:
                store[f"ex_E{t}_{k}"] = factor_matrix(specs2[k], kind)
    store["ex_nterms"] = np.array(op.n_terms)
    store["ex_meta"] = np.array([9, 3.0, 1e-2, 3, 1e-8])
    np.savez_compressed(OUT / "complex.npz", **store)


GENERATORS = {"cp_als": lambda: gen_cp_als(), "ht": lambda: gen_ht(), "operators": lambda: gen_operators(),
              "explicit": lambda: gen_explicit(), "implicit": lambda: gen_implicit(), "io": lambda: gen_io(),
              "diagnostics": lambda: gen_diagnostics(), "complex": lambda: gen_complex(),
              "implicit_forced": lambda: gen_implicit_forced(), "ht_trees": lambda: gen_ht_trees()}


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(GENERATORS)):
        GENERATORS[name]()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
