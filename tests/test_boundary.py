"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/tpde_b200.h declares (no compute calls), and host-side
validation mirrors the reference's error behaviour."""


import numpy as np
import pytest

from paper_1803_10270_b200 import _lib, basis, cp, operators


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = _lib.header_symbols()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n
    assert L.tp_version().decode().startswith("tpde_b200")
    assert L.tp_status_string(0).decode() == "ok"


def test_signatures_cover_header():
    assert set(_lib.header_symbols()) == set(_lib._SIGNATURES)


def test_invalid_arguments_rejected_without_gpu():
    L = _lib.lib()
    q = _lib.int_array([4, 4])
    assert L.tp_cp_inner_f64(0, q, 1, None, 1, None, 0, None, None, 0, None) == _lib.TP_EINVAL
    assert L.tp_cp_als_f64(2, q, 4, None, 2, None, 1, 1e-10, 0, 0.0, 0.0, None, None, 0, None, 0,
                           None) == _lib.TP_EINVAL
    assert L.tp_cp_als_ws_bytes(2, q, 4, 40, 0) > 0    # r > 32: the streamed generic variant
    assert L.tp_cp_als_ws_bytes(2, q, 4, 200, 0) == 0  # r > 160 unsupported


def test_cptensor_validation_mirrors_reference():
    S = (basis.BasisSpec(5, 1.5), basis.BasisSpec(7, 2.0), basis.BasisSpec(3, 0.8))
    with pytest.raises(ValueError, match="one factor matrix per dimension"):
        cp.CPTensor(S, [np.zeros((5, 1))] * 2)
    with pytest.raises(ValueError, match="inconsistent ranks"):
        cp.CPTensor(S, [np.zeros((5, 1)), np.zeros((7, 2)), np.zeros((3, 1))])
    with pytest.raises(ValueError, match="rows != Q"):
        cp.CPTensor(S, [np.zeros((4, 1)), np.zeros((7, 1)), np.zeros((3, 1))])
    # complex factors select the complex128 path; real-valued complex
    # arrays stay on the real fp64 path (the reference's coercion is value-preserving)
    import torch
    assert cp._as_array(np.ones((5, 1)) * 1j, 0).dtype == torch.complex128
    assert cp._as_array(np.ones((5, 1)) + 0j, 0).dtype == torch.float64


def test_basis_spec_rules():
    with pytest.raises(ValueError, match="odd"):
        basis.BasisSpec(4, 1.0)
    basis.BasisSpec(4, 1.0, "collocation")
    with pytest.raises(ValueError, match="b must be positive"):
        basis.BasisSpec(5, 0.0)


def test_fourier_diff_matrix_exact_on_trig():
    for Q in (8, 9, 32):
        x = 2 * np.pi * np.arange(Q) / Q
        D = basis.fourier_diff_matrix(Q)
        for kk in range(1, (Q - 1) // 2 + 1):
            np.testing.assert_allclose(D @ np.sin(kk * x), kk * np.cos(kk * x), atol=1e-11)


def test_operator_validation_and_pairs():
    S = tuple(basis.BasisSpec(6, np.pi, "collocation") for _ in range(3))
    with pytest.raises(ValueError, match="one weight per term"):
        operators.SeparableOperator(S, (1.0,), ((None,) * 3, (None,) * 3))
    with pytest.raises(ValueError, match="at least one term"):
        operators.SeparableOperator(S, (), ())
    with pytest.raises(ValueError, match="every dimension"):
        operators.SeparableOperator(S, (1.0,), ((None,) * 2,))
    L = operators.advection_operator((1.0, 0.5, -0.75), S)
    pair = operators.implicit_euler_pair(L, 0.1)
    assert pair.eta == pytest.approx((1.0, 0.1, 0.05, -0.075), abs=1e-15)
    assert pair.zeta == (1.0, 0.0, 0.0, 0.0)
    cn = operators.crank_nicolson_pair(L, 0.1)
    assert cn.eta[1] == pytest.approx(0.05) and cn.zeta[1] == pytest.approx(-0.05)
    D = operators.dense_factor(basis.BasisSpec(5, 1.0), basis.FactorKind.DERIVATIVE)
    assert D.dtype == np.complex128
    np.testing.assert_allclose(D, np.diag(1j * np.pi * np.arange(-2, 3) / 1.0))   # basis.py:168-187
    with pytest.raises(ValueError, match="complex operator weights"):
        operators.implicit_euler_pair(operators.SeparableOperator(S, (1j,), ((basis.FactorKind.DERIVATIVE, None, None),)),
                                      0.1)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        _lib.device()


def test_explicit_config_validation():
    from paper_1803_10270_b200 import explicit
    with pytest.raises(ValueError, match="dt"):
        explicit.ExplicitConfig(dt=0.0, r_max=2)
    with pytest.raises(ValueError, match="rank cap"):
        explicit.ExplicitConfig(dt=0.1, r_max=0)
    with pytest.raises(ValueError, match="format"):
        explicit.ExplicitConfig(dt=0.1, r_max=2, format="tucker")
    with pytest.raises(ValueError, match="startup"):
        explicit.ExplicitConfig(dt=0.1, r_max=2, startup="euler")
    with pytest.raises(ValueError, match="recipe"):
        explicit.ExplicitConfig(dt=0.1, r_max=2, recipe="magic")


def test_bgk_projection_is_exact_on_grid():
    from paper_1803_10270_b200 import workloads
    W, M, v, w = workloads.bgk_operator_terms(8, 10)
    assert len(W) == 24
    Pv = None
    for wt, row in zip(W[4:], M[4:]):
        t = wt * np.kron(np.kron(row[3], row[4]), row[5])
        Pv = t if Pv is None else Pv + t
    assert np.abs(Pv @ Pv - Pv).max() < 1e-13
    M1 = workloads.maxwellian_1d(v)
    mv = np.kron(np.kron(M1, M1), M1)
    assert np.abs(Pv @ mv - mv).max() < 1e-13


def test_implicit_rejects_complex_galerkin_tables():
    """The reference's Fourier Galerkin pair tables are complex bilinear forms
    (basis.py:207-214); the real-fp64 implicit step must refuse them up front
    instead of reinterpreting complex buffers."""
    from paper_1803_10270_b200 import implicit
    S = tuple(basis.BasisSpec(5, 1.0) for _ in range(3))
    pair = operators.implicit_euler_pair(operators.advection_operator((1.0, 0.5, -0.75), S), 0.1)
    with pytest.raises(ValueError, match="Fourier Galerkin"):
        implicit.build_tables(pair)
    Sc = tuple(basis.BasisSpec(6, np.pi, "collocation") for _ in range(3))
    Dc = np.eye(6) * 1j
    Lc = operators.SeparableOperator(Sc, (1.0,), ((Dc, None, None),))
    with pytest.raises(ValueError, match="complex factor matrices"):
        implicit.build_tables(operators.implicit_euler_pair(Lc, 0.1))


@pytest.mark.gpu
def test_integration_binding_runs():
    """The reference-side ctypes binding printed in INTEGRATION.md, executed as written against a
    stand-in `tensorpde.cp` (the reference's dataclasses by field name: cp.py:38-76, 150-164; the
    reference itself does not travel to the GPU box) and checked against the oracle under the
    reference's trace-scaled regulariser (cp.py:171-173)."""
    import dataclasses
    import re
    import sys
    import types
    from pathlib import Path

    import numpy as np

    from oracle import cp_als as ocp, metrics

    text = (Path(__file__).resolve().parents[1] / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n(# tensorpde/_b200\.py.*?)```", text, re.S).group(1)

    @dataclasses.dataclass(frozen=True)
    class Spec:
        Q: int

    @dataclasses.dataclass
    class CPTensor:
        specs: tuple
        factors: list

        @property
        def ndim(self):
            return len(self.factors)

        @property
        def rank(self):
            return self.factors[0].shape[1]

    @dataclasses.dataclass(frozen=True)
    class ALSApproxConfig:
        max_sweeps: int = 200
        tol: float = 0.0
        stall: float = 1e-13
        seed: int = 0
        quad_points: int = 0

    class ConditioningError(RuntimeError):
        pass

    def random_cp(specs, r, rng):
        return CPTensor(specs, [rng.standard_normal((s.Q, r)).astype(complex) for s in specs])

    ref_cp = types.ModuleType("tensorpde.cp")
    ref_cp.CPTensor, ref_cp.ALSApproxConfig = CPTensor, ALSApproxConfig
    ref_cp.ConditioningError, ref_cp.random_cp = ConditioningError, random_cp
    pkg = types.ModuleType("tensorpde")
    pkg.cp = ref_cp
    saved = {k: sys.modules.get(k) for k in ("tensorpde", "tensorpde.cp")}
    sys.modules["tensorpde"], sys.modules["tensorpde.cp"] = pkg, ref_cp
    try:
        ns = {}
        exec(compile(code, "INTEGRATION.md", "exec"), ns)
        rng = np.random.default_rng(3)
        qs, R, r = (14, 11, 12), 9, 3
        specs = tuple(Spec(q) for q in qs)
        V = [rng.standard_normal((q, R)) for q in qs]
        init = [v[:, :r].copy() for v in V]
        trace = []
        out = ns["cp_approx_als"](CPTensor(specs, [v.astype(complex) for v in V]), r,
                                  ALSApproxConfig(max_sweeps=7, stall=-np.inf),
                                  init=CPTensor(specs, [u.astype(complex) for u in init]), trace=trace)
        otrace = []
        ref = ocp.als(V, init, 7, lam=None, trace=otrace)
        assert metrics.cp_rel_diff(ref, [f.real for f in out.factors]) <= 1e-9
        np.testing.assert_allclose(trace, otrace, rtol=1e-8, atol=1e-12)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
