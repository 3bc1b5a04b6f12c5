"""Pin the CPU oracle against golden vectors produced by the live reference
(oracle/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import unso_oracle as O


def _kw(name, kats):
    return dict(
        unso_default=dict(method="unso"),
        unso_generic=dict(method="unso", a=kats["kat"]["generic_a"], rule="approx-abs"),
        unso_plain=dict(method="unso", scaling="plain"),
        unso_gelfand=dict(method="unso", scaling="gelfand"),
        original4=dict(method="original", iterations=4),
        muon3=dict(method="muon", iterations=3),
        muon5=dict(method="muon", iterations=5),
        cesista=dict(method="cesista", rows=O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES)),
        external=dict(method="external", rows=O.muon_rows(3)),
    )[name]


def test_rng_words_bit_exact(golden_kats):
    k = golden_kats["kat"]
    assert [int(v) for v in O.stream_words(0, 0, 8)] == k["rng_words_seed0"]
    assert [int(v) for v in O.stream_words(7, 5, 4)] == k["rng_words_seed7_start5"]
    assert O.stream_normals(3, 0, 7).tolist() == k["rng_normals_seed3"]


def test_cfg1_input_bit_exact(golden_kats):
    g = O.gaussian_matrix(512, 128, 0)
    assert hashlib.sha256(np.ascontiguousarray(g).tobytes()).hexdigest() == golden_kats["kat"]["cfg1_input_sha256"]


def test_final_coefficient_kats(golden_kats):
    k = golden_kats["kat"]
    assert O.final_coefficient(14, O.DEFAULT_A, "exact") == k["derive_b_default"]
    assert O.final_coefficient(14, O.DEFAULT_A, "exact") == pytest.approx(211.85214059820694, abs=1e-9)
    assert O.final_coefficient(1, [], "exact") == pytest.approx(1.0980762113533158, abs=1e-12)
    assert O.final_coefficient(14, np.zeros(13), "approx-sum") == pytest.approx(209.3876013789163, abs=1e-9)
    assert O.final_coefficient(14, k["generic_a"], "approx-abs") == k["derive_b_generic_abs"]


def test_poly_value_and_scalar_maps(golden_kats):
    k = golden_kats["kat"]
    grid = np.array(k["eval_f_grid"])
    np.testing.assert_array_equal(O.poly_value(14, O.DEFAULT_A, "exact", grid), np.array(k["eval_f_default"]))
    maps = k["scalar_maps"]
    np.testing.assert_array_equal(O.composed_map("unso")(grid), maps["unso"])
    np.testing.assert_array_equal(O.composed_map("original")(grid), maps["original8"])
    np.testing.assert_array_equal(O.composed_map("muon")(grid), maps["muon5"])
    np.testing.assert_array_equal(O.composed_map("cesista", rows=O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES))(grid),
                                  maps["cesista"])


def test_flop_model(golden_kats):
    rows = O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES)
    for shape, d in golden_kats["kat"]["flops"].items():
        h, w = map(int, shape.split("x"))
        assert O.model_flops("unso", h, w) == d["unso"]
        assert O.model_flops("original", h, w) == d["original8"]
        assert O.model_flops("muon", h, w) == d["muon5"]
        assert O.model_flops("cesista", h, w, rows=rows) == d["cesista"]


def test_small_cases_match_reference(golden_arrays, golden_kats):
    worst = 0.0
    for case in golden_kats["cases"]:
        out = O.run(golden_arrays[case["input"]], **_kw(case["method"], golden_kats))
        ref = golden_arrays["y_" + case["key"]]
        worst = max(worst, float(np.max(np.abs(out["y"] - ref))))
        assert out["flops"] == case["flops"]
        assert out["preprocess_flops"] == case["preprocess_flops"]
        assert out["was_transposed"] == case["was_transposed"]
        assert [list(s) for s in out["shapes"]] == case["shapes"]
        assert O.ortho_error_any(out["y"]) == pytest.approx(case["ortho_error"], rel=1e-10, abs=1e-12)
    assert worst <= 1e-12


def test_cfg1_outputs_match_reference(golden_arrays, golden_kats):
    g = O.gaussian_matrix(512, 128, 0)
    m32 = g.astype(np.float32).astype(np.float64)
    out = O.run(m32, "unso")
    np.testing.assert_allclose(out["y"], golden_arrays["cfg1_fp32_unso"], rtol=0, atol=1e-12)
    assert O.ortho_error_any(out["y"]) == pytest.approx(0.038734205096269951, rel=1e-9)
    mu = O.run(m32, "muon", iterations=5)
    np.testing.assert_allclose(mu["y"], golden_arrays["cfg1_fp32_muon5"], rtol=0, atol=1e-12)
    assert golden_kats["cfg1"]["fp32_muon5"]["ortho_error"] == pytest.approx(4.322727279270854, rel=1e-9)


def test_long_side_economy():
    """UNSO touches the long side exactly twice for any order (tests/test_ortho.py:104-110)."""
    x = O.gaussian_matrix(32, 96, 1)
    for order in (2, 8, 14):
        log = O.ContractionLog()
        xs, _, _ = O.scale_and_orient(x, "gram")
        O.unso_poly(xs, order, np.full(order - 1, 0.3), "approx-abs", log)
        assert sum(1 for s in log.shapes if 96 in s) == 2


def test_degenerate_and_shape_errors():
    with pytest.raises(ValueError, match="degenerate"):
        O.run(np.zeros((4, 8)), "unso")
    with pytest.raises(ValueError, match="shape"):
        O.unso_poly(np.ones((4, 2)))


def test_sampled_restatements_match_the_full_oracle():
    """unso_sampled / quintic_sampled (long-side samples for full-size GPU parity) equal the
    op-for-op oracle on tall, wide and square inputs."""
    rng = np.random.default_rng(3)
    for shape in ((96, 40), (40, 96), (50, 50)):
        m = rng.standard_normal(shape)
        long = max(shape)
        idx = np.sort(rng.choice(long, 17, replace=False))
        tall = shape[0] > shape[1]
        for scaling in ("gram", "plain"):
            full = O.run(m, "unso", scaling=scaling)["y"]
            got = O.unso_sampled(m, idx, scaling=scaling)
            want = full[idx] if tall else full[:, idx]
            assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), (shape, scaling)
        full = O.run(m, "muon", iterations=5)["y"]
        got = O.quintic_sampled(m, idx)
        want = full[idx] if tall else full[:, idx]
        assert np.abs(got - want).max() <= 1e-11 * max(1.0, np.abs(want).max()), shape
