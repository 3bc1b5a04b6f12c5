"""Host-side logic of the product package (no GPU): coefficient handling,
MethodSpec validation, FLOP model and scalar maps, checked against the
reference's golden vectors."""

import numpy as np
import pytest

import paper_2602_02500_b200 as U
from paper_2602_02500_b200.errors import ParseError


def test_default_coefficients_match_reference(golden_kats):
    c = U.default_coefficients()
    assert c.order == 14 and c.b_rule is U.BRule.EXACT
    assert U.derive_b(c) == golden_kats["kat"]["derive_b_default"]
    dc = c.device_coefficients()
    assert dc.shape == (14,) and dc[-1] == U.derive_b(c)


def test_derive_b_rules(golden_kats):
    k = golden_kats["kat"]
    assert U.derive_b(U.CoefficientSet(1, np.zeros(0), "exact")) == pytest.approx(1.0980762113533158, abs=1e-12)
    assert U.derive_b(U.CoefficientSet(14, np.zeros(13), "approx-sum")) == pytest.approx(209.3876013789163, abs=1e-9)
    assert U.derive_b(U.CoefficientSet(14, np.array(k["generic_a"]), "approx-abs")) == k["derive_b_generic_abs"]
    assert abs(U.constraint_residual(U.default_coefficients())) < 1e-9


def test_eval_f_and_scalar_maps(golden_kats):
    k = golden_kats["kat"]
    grid = np.array(k["eval_f_grid"])
    np.testing.assert_array_equal(U.eval_f(U.default_coefficients(), grid), k["eval_f_default"])
    ces = U.CesistaStepParams(U.default_cesista_triples())
    specs = {
        "unso": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()),
        "original8": U.MethodSpec(U.MethodKind.ORIGINAL_NS),
        "muon5": U.MethodSpec(U.MethodKind.MUON_NS),
        "cesista": U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=ces),
    }
    for name, spec in specs.items():
        np.testing.assert_array_equal(U.scalar_map(spec)(grid), k["scalar_maps"][name])


def test_kernel_model_flops(golden_kats):
    ces = U.CesistaStepParams(U.default_cesista_triples())
    specs = {
        "unso": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()),
        "original8": U.MethodSpec(U.MethodKind.ORIGINAL_NS),
        "muon5": U.MethodSpec(U.MethodKind.MUON_NS),
        "cesista": U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=ces),
    }
    for shape, d in golden_kats["kat"]["flops"].items():
        h, w = map(int, shape.split("x"))
        for name, spec in specs.items():
            assert U.kernel_model_flops(h, w, spec) == d[name], (shape, name)


def test_model_shapes_and_preprocess_flops(golden_kats):
    """The contraction audit and preprocess FLOPs equal the reference's counters."""
    for case in golden_kats["cases"]:
        r, c = map(int, case["input"][3:].split("x"))
        h, w = min(r, c), max(r, c)
        if r == c:
            h, w = r, c
        name = case["method"]
        spec = {
            "unso_default": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()),
            "unso_generic": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.CoefficientSet(
                14, np.array(golden_kats["kat"]["generic_a"]), "approx-abs")),
            "unso_plain": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="plain"),
            "unso_gelfand": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="gelfand"),
            "original4": U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=4),
            "muon3": U.MethodSpec(U.MethodKind.MUON_NS, iterations=3),
            "muon5": U.MethodSpec(U.MethodKind.MUON_NS, iterations=5),
            "cesista": U.MethodSpec(U.MethodKind.CESISTA_NS,
                                    step_params=U.CesistaStepParams(U.default_cesista_triples())),
            "external": U.MethodSpec(U.MethodKind.EXTERNAL_SCHEDULE,
                                     schedule=np.tile(np.array(U.MUON_COEFFICIENTS), (3, 1))),
        }[name]
        assert U.kernel_model_flops(h, w, spec) == case["flops"], case["key"]
        assert [list(s) for s in U.model_matmul_shapes(h, w, spec)] == case["shapes"], case["key"]
        assert U.preprocess_model_flops(h, w, spec.effective_scaling, spec.gelfand_power) == \
            case["preprocess_flops"], case["key"]


def test_unso_long_side_products_two_for_any_order():
    for order in (2, 8, 14):
        spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.CoefficientSet(order, np.full(order - 1, 0.3)))
        shapes = U.executed_matmul_shapes(32, 96, spec)
        assert sum(1 for s in shapes if 96 in s) == 2
    muon = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)
    assert sum(1 for s in U.executed_matmul_shapes(32, 96, muon) if 96 in s) == 10


def test_method_spec_validation():
    assert U.MethodSpec(U.MethodKind.ORIGINAL_NS).iterations == 8
    assert U.MethodSpec(U.MethodKind.MUON_NS).iterations == 5
    assert U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()).effective_scaling is U.Scaling.FROBENIUS_GRAM
    assert U.MethodSpec(U.MethodKind.MUON_NS).effective_scaling is U.Scaling.FROBENIUS_PLAIN
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.UNSO)
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.MUON_NS, iterations=0)
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.CESISTA_NS)
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.EXTERNAL_SCHEDULE, schedule=np.zeros((2, 2)))
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), precision="fp8")
    with pytest.raises(ValueError):
        U.CoefficientSet(3, np.array([1.0, np.inf]))
    # recipe knobs of this implementation (not in the reference): validated the same way
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, ns_products="fp8")
    with pytest.raises(ValueError):
        U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), chain="fp8")
    from paper_2602_02500_b200 import _native as N
    from paper_2602_02500_b200.ortho import Precision, _build_method_desc
    md, _ = _build_method_desc(U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, ns_products="bf16"), Precision.BF16, 1)
    assert md.flags & N.FLAG_NS_SINGLE_STATE
    md, _ = _build_method_desc(U.MethodSpec(U.MethodKind.MUON_NS, iterations=5), Precision.BF16, 1)
    assert not md.flags & N.FLAG_NS_SINGLE_STATE


def test_expand_cesista_rows():
    rows = U.expand_cesista_rows(np.array([[1.0, 0.0, 0.0]]))
    np.testing.assert_allclose(rows, [[2.0, -2.0, 1.0]], atol=1e-15)


def test_coefficient_file_round_trip(tmp_path):
    c = U.default_coefficients()
    p = tmp_path / "c.txt"
    U.write_coefficients(p, c)
    back = U.read_coefficients(p)
    assert back.order == c.order and back.b_rule == c.b_rule
    np.testing.assert_array_equal(back.a, c.a)
    bad = tmp_path / "bad.txt"
    bad.write_text("3 nope\n1\n2\n")
    with pytest.raises(ParseError):
        U.read_coefficients(bad)
    bad.write_text("3 exact\n1\n")
    with pytest.raises(ParseError):
        U.read_coefficients(bad)


def test_step_triples_reader(tmp_path):
    p = tmp_path / "s.txt"
    p.write_text("1 2 3\n4 5 6\n")
    np.testing.assert_array_equal(U.read_step_triples(p), [[1, 2, 3], [4, 5, 6]])
    p.write_text("1 2\n")
    with pytest.raises(ParseError):
        U.read_step_triples(p)
