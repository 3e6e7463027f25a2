"""GPU parity of the implicit ALS step (implicit.step, implicit.py:222-301) against
the oracle (pinned by tests/golden/implicit.npz, which ran the real reference with
SURVEY shims S5-S8), in both gamma orientations."""

import math

import numpy as np
import pytest

from conftest import load_golden, unpack_cp
from oracle import implicit as oim
from oracle import metrics

pytestmark = pytest.mark.gpu

from paper_1803_10270_b200 import cp, implicit, operators, workloads  # noqa: E402
from paper_1803_10270_b200.basis import BasisSpec, fourier_diff_matrix  # noqa: E402


def col_specs(d, q):
    return tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for _ in range(d))


def euler_pair(S, D, a, dt):
    d = len(S)
    L = operators.SeparableOperator(S, tuple(-np.asarray(a)), tuple(tuple(D if k == t else None for k in range(d))
                                                                  for t in range(d)))
    return operators.implicit_euler_pair(L, dt)


def oracle_tables(d, q, D, a, dt):
    mats = [[None] * d] + [[D if k == i else None for k in range(d)] for i in range(d)]
    eta = [1.0] + list(dt * np.asarray(a))
    zeta = [1.0] + [0.0] * d
    return oim.build_tables(mats, eta, zeta, [q] * d)


@pytest.mark.parametrize("orientation,key", [("reference", "out_reference_orientation"),
                                             ("corrected", "out_corrected")])
def test_step_golden(orientation, key):
    g = load_golden("implicit")
    q, d, r, dt, sweeps, lam = g["meta"]
    q, d, sweeps = int(q), int(d), int(sweeps)
    S = col_specs(d, q)
    pair = euler_pair(S, g["D"], g["a"], float(dt))
    cfg = implicit.ALSStepConfig(dt=float(dt), eps_tol=0.0, max_sweeps=sweeps, delta_beta=1.0,
                                 schedule="gauss-seidel", lam=float(lam), orientation=orientation)
    log = {}
    out = implicit.step(cp.CPTensor(S, unpack_cp(g, "f0")), pair, None, cfg, log=log)
    assert log["sweeps"] == sweeps
    rel = metrics.cp_rel_diff(unpack_cp(g, key), out.to_numpy())
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("solver", ["dense", "circulant"])
@pytest.mark.parametrize("schedule,delta", [("gauss-seidel", 1.0), ("jacobi", 4.0), ("jacobi", 1.0)])
def test_step_matches_oracle(schedule, delta, solver):
    rng = np.random.default_rng(7)
    d, q, r, dt, sweeps = 4, 16, 4, 2e-2, 5
    a = (1.0, 0.5, -0.75, 0.25)
    D = fourier_diff_matrix(q)
    S = col_specs(d, q)
    f0 = [rng.standard_normal((q, r)) for _ in range(d)]
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=delta, schedule=schedule,
                                 lam=1e-10, solver=solver)
    out = implicit.step(cp.CPTensor(S, f0), euler_pair(S, D, a, dt), None, cfg)
    ref, done, _ = oim.step(f0, oracle_tables(d, q, D, a, dt), sweeps, 1e-10, schedule=schedule,
                            delta_beta=delta)
    rel = metrics.cp_rel_diff(ref, out.to_numpy())
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("solver", ["dense", "circulant"])
def test_config2_full_size_step(solver):
    """BASELINE config 2 sizes (d=6, Q=128, r=16 -> 2048^2 normal equations), 3 sweeps
    of one step, vs the oracle's direct solves (dense Cholesky and DFT-block paths)."""
    w = workloads.cfg2(0)
    S, D, a, dt = w["specs"], w["D"], w["a"], w["dt"]
    f0 = w["ic"]["factors"]
    sweeps = 3
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=1.0, schedule="gauss-seidel",
                                 lam=w["lam"], solver=solver)
    out = implicit.step(cp.CPTensor(S, f0), euler_pair(S, D, a, dt), None, cfg)
    ref, _, _ = oim.step(f0, oracle_tables(6, 128, D, a, dt), sweeps, w["lam"])
    rel = metrics.cp_rel_diff(ref, out.to_numpy())
    assert rel <= 1e-8, rel


def test_dense_cholesky_blocked():
    """Dense solver: blocked Cholesky (left-looking diagonal blocks) with the lower-tile SYRK
    and the multi-CTA block solves on a system of several 64-blocks (r Q = 6 x 48 = 288 ->
    padded 320), vs the oracle."""
    if True:
        rng = np.random.default_rng(17)
        d, q, r, dt, sweeps = 3, 48, 6, 2e-2, 3
        a = (1.0, -0.5, 0.75)
        D = fourier_diff_matrix(q)
        S = col_specs(d, q)
        f0 = [rng.standard_normal((q, r)) for _ in range(d)]
        cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=1.0,
                                     schedule="gauss-seidel", lam=1e-10, solver="dense")
        out = implicit.step(cp.CPTensor(S, f0), euler_pair(S, D, a, dt), None, cfg)
        ref, _, _ = oim.step(f0, oracle_tables(d, q, D, a, dt), sweeps, 1e-10)
        assert metrics.cp_rel_diff(ref, out.to_numpy()) <= 1e-9


@pytest.mark.parametrize("schedule,delta", [("gauss-seidel", 1.0), ("jacobi", 4.0)])
def test_step_nonuniform_mode_sizes(schedule, delta):
    """Modes of different sizes (Q = 12, 20, 9, 16): zero-padded tables and states inside
    implicit.step (the padding rows decouple and stay zero), vs the oracle on the true sizes."""
    rng = np.random.default_rng(23)
    qs, r, dt, sweeps = (12, 20, 9, 16), 4, 2e-2, 4
    a = (1.0, 0.5, -0.75, 0.25)
    d = len(qs)
    S = tuple(BasisSpec(q, math.pi, "collocation", lo=0.0) for q in qs)
    Ds = [fourier_diff_matrix(q) for q in qs]
    L = operators.SeparableOperator(S, tuple(-np.asarray(a)),
                                    tuple(tuple(Ds[k] if k == t else None for k in range(d)) for t in range(d)))
    pair = operators.implicit_euler_pair(L, dt)
    f0 = [rng.standard_normal((q, r)) for q in qs]
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=delta, schedule=schedule,
                                 lam=1e-10)
    out = implicit.step(cp.CPTensor(S, f0), pair, None, cfg)
    assert out.qs == qs
    mats = [[None] * d] + [[Ds[k] if k == i else None for k in range(d)] for i in range(d)]
    tabs = oim.build_tables(mats, [1.0] + list(dt * np.asarray(a)), [1.0] + [0.0] * d, list(qs))
    ref, _, _ = oim.step(f0, tabs, sweeps, 1e-10, schedule=schedule, delta_beta=delta)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= 1e-9


def test_config_validation():
    with pytest.raises(ValueError, match="schedule"):
        implicit.ALSStepConfig(dt=0.1, schedule="sor")
    with pytest.raises(ValueError, match="damping"):
        implicit.ALSStepConfig(dt=0.1, delta_beta=0.5)


def test_config2_trajectory_circulant_vs_dense():
    """Several full 20-sweep steps at config-2 sizes: DFT-block path vs dense Cholesky
    path vs oracle after 2 steps (final-solution bar 1e-8)."""
    w = workloads.cfg2(0)
    S, D, a, dt = w["specs"], w["D"], w["a"], w["dt"]
    f0 = w["ic"]["factors"]
    pair = euler_pair(S, D, a, dt)
    outs = {}
    for solver in ("circulant", "dense"):
        cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=w["sweeps"], delta_beta=1.0,
                                     schedule="gauss-seidel", lam=w["lam"], solver=solver)
        outs[solver] = implicit.run(cp.CPTensor(S, f0), pair, cfg, 2).to_numpy()
    tab = oracle_tables(6, 128, D, a, dt)
    ref = f0
    for _ in range(2):
        ref, _, _ = oim.step(ref, tab, w["sweeps"], w["lam"])
    for solver, out in outs.items():
        assert metrics.cp_rel_diff(ref, out) <= 1e-8, solver


def test_circulant_detection():
    from paper_1803_10270_b200.basis import fourier_diff_matrix as fdm
    assert implicit.is_circulant(fdm(16))
    assert implicit.is_circulant(fdm(16).T @ fdm(16))
    assert not implicit.is_circulant(np.diag(np.arange(8.0)))


@pytest.fixture
def circ_fused():
    import ctypes
    from paper_1803_10270_b200 import _lib
    L = _lib.lib()
    L.tp_debug_set_circ_fused.argtypes = [ctypes.c_int]
    yield L.tp_debug_set_circ_fused
    L.tp_debug_set_circ_fused(1)


@pytest.mark.parametrize("fused", [0, 1])
@pytest.mark.parametrize("orientation", ["corrected", "reference"])
@pytest.mark.parametrize("d,q,r,eps_tol", [(3, 15, 5, 1e-7), (4, 16, 4, 0.0), (2, 9, 3, 1e-4)])
def test_circulant_gauss_seidel_fused(circ_fused, fused, orientation, d, q, r, eps_tol):
    """Fused one-launch circulant Gauss-Seidel step (half spectrum kept on the device)
    and the per-kernel path against the oracle: odd and even Q, early stop on eps_tol
    (same sweep count as the reference loop, implicit.py:244), both gamma orientations."""
    circ_fused(fused)
    rng = np.random.default_rng(40 + q)
    dt, sweeps = 2e-2, 30
    a = tuple(rng.uniform(-1, 1, d))
    D = fourier_diff_matrix(q)
    S = col_specs(d, q)
    f0 = [rng.standard_normal((q, r)) for _ in range(d)]
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=eps_tol, max_sweeps=sweeps if eps_tol > 0 else 6, delta_beta=1.0,
                                 schedule="gauss-seidel", lam=1e-10, solver="circulant", orientation=orientation)
    log = {}
    out = implicit.step(cp.CPTensor(S, f0), euler_pair(S, D, a, dt), None, cfg, log=log)
    ref, done, eps = oim.step(f0, oracle_tables(d, q, D, a, dt), cfg.max_sweeps, 1e-10, eps_tol=eps_tol,
                              orientation=orientation)
    assert log["sweeps"] == done
    assert abs(log["eps_conv"] - eps) <= 1e-8 * max(eps, 1e-300) + 1e-14
    rel = metrics.cp_rel_diff(ref, out.to_numpy())
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("fused", [0, 1])
def test_config2_steps_fused_vs_unfused(circ_fused, fused):
    """Config-2 sizes, 2 full steps of 20 sweeps, both circulant paths vs the oracle."""
    circ_fused(fused)
    w = workloads.cfg2(0)
    S, D, a, dt = w["specs"], w["D"], w["a"], w["dt"]
    f0 = w["ic"]["factors"]
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=w["sweeps"], delta_beta=1.0,
                                 schedule="gauss-seidel", lam=w["lam"], solver="circulant")
    out = implicit.run(cp.CPTensor(S, f0), euler_pair(S, D, a, dt), cfg, 2).to_numpy()
    tab = oracle_tables(6, 128, D, a, dt)
    ref = f0
    for _ in range(2):
        ref, _, _ = oim.step(ref, tab, w["sweeps"], w["lam"])
    assert metrics.cp_rel_diff(ref, out) <= 1e-8


@pytest.mark.parametrize("solver", ["dense", "circulant"])
@pytest.mark.parametrize("case", ["gs", "jac"])
@pytest.mark.parametrize("orientation,key", [("reference", "out_reference_orientation"),
                                             ("corrected", "out_corrected")])
def test_forced_step_golden(solver, case, orientation, key):
    """Forced implicit steps of the real reference (tests/golden/implicit_forced.npz,
    forcing block implicit.py:140-152): Gauss-Seidel with fixed sweeps, and the
    default Jacobi schedule (delta_beta = 4) whose eps_tol stop is decided on the
    device -- the sweep count must equal the reference's."""
    g = load_golden("implicit_forced")
    q, d, r, dt, lam = g["meta"]
    q, d = int(q), int(d)
    eps_tol, max_sweeps, delta_beta, jac = g[f"{case}_cfg"]
    S = col_specs(d, q)
    pair = euler_pair(S, g["D"], g["a"], float(dt))
    cfg = implicit.ALSStepConfig(dt=float(dt), eps_tol=float(eps_tol), max_sweeps=int(max_sweeps),
                                 delta_beta=float(delta_beta), schedule="jacobi" if jac else "gauss-seidel",
                                 lam=float(lam), orientation=orientation, solver=solver)
    log = {}
    out = implicit.step(cp.CPTensor(S, unpack_cp(g, "f0")), pair, cp.CPTensor(S, unpack_cp(g, "forcing")), cfg,
                        log=log)
    idx = 0 if orientation == "reference" else 1
    assert log["sweeps"] == int(g[f"{case}_sweeps"][idx])
    assert log["lsqr_iterations"] is None and log["solve_seconds"] > 0
    rel = metrics.cp_rel_diff(unpack_cp(g, f"{case}_{key}"), out.to_numpy())
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("solver", ["dense", "circulant"])
def test_forced_step_matches_oracle_larger(solver):
    rng = np.random.default_rng(17)
    d, q, r, rf, dt, sweeps = 4, 16, 4, 3, 2e-2, 6
    a = (1.0, 0.5, -0.75, 0.25)
    D = fourier_diff_matrix(q)
    S = col_specs(d, q)
    f0 = [rng.standard_normal((q, r)) for _ in range(d)]
    c = [0.3 * rng.standard_normal((q, rf)) for _ in range(d)]
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=0.0, max_sweeps=sweeps, delta_beta=1.0, schedule="gauss-seidel",
                                 lam=1e-10, solver=solver)
    out = implicit.step(cp.CPTensor(S, f0), euler_pair(S, D, a, dt), cp.CPTensor(S, c), cfg)
    ref, _, _ = oim.step(f0, oracle_tables(d, q, D, a, dt), sweeps, 1e-10, forcing=c, dt=dt)
    assert metrics.cp_rel_diff(ref, out.to_numpy()) <= 1e-9


def test_implicit_run_is_stream_ordered_and_capturable():
    """No host synchronisation inside implicit.step's launch: with eps_tol > 0 (the
    device-side stop) the dense path can be captured in a CUDA graph and replayed,
    bitwise equal to eager."""
    import torch
    rng = np.random.default_rng(23)
    d, q, r, dt = 3, 12, 3, 2e-2
    a = (1.0, 0.5, -0.75)
    S = col_specs(d, q)
    D = fourier_diff_matrix(q)
    pair = euler_pair(S, D, a, dt)
    cfg = implicit.ALSStepConfig(dt=dt, eps_tol=1e-4, max_sweeps=200, delta_beta=4.0, schedule="jacobi",
                                 lam=1e-10, solver="dense")
    ws = implicit.StepWorkspace(pair, cfg)
    f0 = cp.CPTensor(S, [rng.standard_normal((q, r)) for _ in range(d)])
    eager = implicit.run(f0, pair, cfg, 2, workspace=ws)
    out = f0.data.clone()
    eps = torch.zeros(1, dtype=torch.float64, device=out.device)
    info = torch.zeros(2, dtype=torch.int32, device=out.device)
    implicit._launch(f0, out, ws.tables, cfg, eps, info)      # warm-up: tables cached, workspace sized
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            out.copy_(f0.data)
            implicit._launch(f0, out, ws.tables, cfg, eps, info)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    one = implicit.run(f0, pair, cfg, 1, workspace=ws)
    assert torch.equal(out, one.data)
    assert 0 < int(info[1].item()) < 200      # stopped on the device by eps_tol
    assert eager.data.shape == one.data.shape
