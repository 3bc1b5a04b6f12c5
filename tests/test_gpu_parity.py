"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference's golden vectors.  Tolerances (BASELINE.json north_star):
    fp32 mode  ||Y - Y_ref||_F / ||Y_ref||_F <= 1e-5
    bf16 mode  ... <= 2e-2, the oracle fed the same bf16-rounded input
fp64 inputs run the fp32-mode pipeline end to end in fp64 and must agree with
the reference to 1e-10."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "bf16": 2e-2}
DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).double().numpy()


def spec_for(name, kats):
    ces = U.CesistaStepParams(U.default_cesista_triples())
    return {
        "unso_default": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()),
        "unso_generic": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.CoefficientSet(
            14, np.array(kats["kat"]["generic_a"]), "approx-abs")),
        "unso_plain": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="plain"),
        "unso_gelfand": U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="gelfand"),
        "original4": U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=4),
        "muon3": U.MethodSpec(U.MethodKind.MUON_NS, iterations=3),
        "muon5": U.MethodSpec(U.MethodKind.MUON_NS, iterations=5),
        "cesista": U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=ces),
        "external": U.MethodSpec(U.MethodKind.EXTERNAL_SCHEDULE,
                                 schedule=np.tile(np.array(U.MUON_COEFFICIENTS), (3, 1))),
    }[name]


def oracle_kw(name, kats):
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


def run(m_np, spec, dtype, precision):
    x = torch.from_numpy(np.ascontiguousarray(m_np)).to(DEV, dtype)
    res = U.orthogonalize(x, spec, precision=precision)
    torch.cuda.synchronize()
    return res, res.y.double().cpu().numpy()


# ------------------------------------------------------------------ golden small cases
def test_small_cases_fp64_io_match_reference(golden_arrays, golden_kats):
    """fp64 in/out: the fp32-mode pipeline is fp64 end to end -> 1e-10 against the live reference."""
    worst = 0.0
    for case in golden_kats["cases"]:
        m = golden_arrays[case["input"]]
        res, y = run(m, spec_for(case["method"], golden_kats), torch.float64, "fp32")
        ref = golden_arrays["y_" + case["key"]]
        r = rel(y, ref)
        worst = max(worst, r)
        assert r <= 1e-10, (case["key"], r)
        assert res.flops == case["flops"]
        assert res.was_transposed == case["was_transposed"]
    print(f"worst fp64-io rel err over {len(golden_kats['cases'])} cases: {worst:.2e}")


def test_small_cases_fp32_mode(golden_arrays, golden_kats):
    for case in golden_kats["cases"]:
        m = golden_arrays[case["input"]].astype(np.float32)
        _, y = run(m, spec_for(case["method"], golden_kats), torch.float32, "fp32")
        ref = O.run(m.astype(np.float64), **oracle_kw(case["method"], golden_kats))["y"]
        assert rel(y, ref) <= TOL["fp32"], case["key"]


def test_small_cases_bf16_mode_unso(golden_arrays, golden_kats):
    for case in golden_kats["cases"]:
        if not case["method"].startswith("unso"):
            continue
        m = golden_arrays[case["input"]].astype(np.float32)
        res, y = run(m, spec_for(case["method"], golden_kats), torch.bfloat16, "bf16")
        ref = O.run(bf16_round(m), **oracle_kw(case["method"], golden_kats))["y"]
        r = rel(y, ref)
        assert r <= TOL["bf16"], (case["key"], r)
        assert res.precision == "bf16"


# ------------------------------------------------------------------ cfg1 (BASELINE configs[0])
def test_cfg1_fp32_mode(golden_arrays, golden_kats):
    g = O.gaussian_matrix(512, 128, 0).astype(np.float32)
    for name, spec in (("unso", U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())),
                       ("muon5", U.MethodSpec(U.MethodKind.MUON_NS, iterations=5))):
        res, y = run(g, spec, torch.float32, "fp32")
        ref = golden_arrays[f"cfg1_fp32_{name}"]
        r = rel(y, ref)
        err = U.ortho_error_any(res.y)
        ref_err = golden_kats["cfg1"][f"fp32_{name}"]["ortho_error"]
        print(f"cfg1 {name} fp32: rel {r:.2e}  ortho_error {err:.6f} (reference {ref_err:.6f})")
        assert r <= TOL["fp32"], (name, r)
        assert err == pytest.approx(ref_err, rel=1e-4)


def test_cfg1_bf16_mode(golden_arrays, golden_kats):
    g = O.gaussian_matrix(512, 128, 0).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    for dtype in (torch.bfloat16, torch.float32):
        res, y = run(g, spec, dtype, "bf16")
        r = rel(y, golden_arrays["cfg1_bf16_unso"])
        print(f"cfg1 unso bf16 mode ({dtype}): rel {r:.2e}")
        assert r <= TOL["bf16"]


# ------------------------------------------------------------------ properties (tests/test_ortho.py)
def test_orthonormal_rows_are_a_fixed_point():
    q, _ = np.linalg.qr(O.gaussian_matrix(256, 64, 3))
    x = torch.from_numpy(np.ascontiguousarray(q.T)).to(DEV)
    y = U.unso(x, U.default_coefficients())
    assert torch.allclose(y, x, atol=1e-10)
    y32 = U.unso(x.float(), U.default_coefficients())
    assert rel(y32.double().cpu().numpy(), q.T) <= 1e-5


def test_diagonal_inputs_stay_diagonal():
    d = np.diag([0.9, 0.7, 0.5, 0.3, 0.2])
    for spec in (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()),
                 U.MethodSpec(U.MethodKind.MUON_NS, iterations=3)):
        _, y = run(d, spec, torch.float64, "fp32")
        assert np.max(np.abs(y - np.diag(np.diag(y)))) < 1e-12


def test_zero_matrix_is_degenerate():
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    for dtype, prec in ((torch.float32, "fp32"), (torch.bfloat16, "bf16")):
        with pytest.raises(U.DegenerateInputError):
            U.orthogonalize(torch.zeros(64, 256, device=DEV, dtype=dtype), spec, precision=prec)
    with pytest.raises(U.DegenerateInputError):
        U.orthogonalize(torch.zeros(64, 256, device=DEV), U.MethodSpec(U.MethodKind.MUON_NS))


def test_row_wide_precondition():
    with pytest.raises(U.ShapeError):
        U.unso(torch.ones(4, 2, device=DEV, dtype=torch.float64), U.default_coefficients())


def test_transpose_equivariance():
    m = O.gaussian_matrix(96, 200, 4)
    for spec in (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()),
                 U.MethodSpec(U.MethodKind.MUON_NS, iterations=3)):
        _, a = run(m, spec, torch.float64, "fp32")
        _, b = run(m.T, spec, torch.float64, "fp32")
        assert np.max(np.abs(a - b.T)) < 1e-12


def test_batch_equals_single_calls():
    ms = np.stack([O.gaussian_matrix(384, 128, s) for s in range(3)]).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    for dtype, prec in ((torch.float32, "fp32"), (torch.bfloat16, "bf16")):
        xb = torch.from_numpy(ms).to(DEV, dtype)
        yb = U.orthogonalize(xb, spec, precision=prec).y
        for i in range(3):
            yi = U.orthogonalize(xb[i], spec, precision=prec).y
            r = rel(yb[i].double().cpu().numpy(), yi.double().cpu().numpy())
            assert r <= (1e-6 if prec == "fp32" else 1e-2), (prec, i, r)


def test_ortho_error_device_matches_oracle():
    y = O.gaussian_matrix(300, 70, 9) * 0.1
    got = U.ortho_error_any(torch.from_numpy(y).to(DEV))
    assert got == pytest.approx(O.ortho_error_any(y), rel=1e-12)


def test_preprocess_and_bare_kernels_match_oracle():
    m = O.gaussian_matrix(160, 48, 12)
    x, tall = U.preprocess(torch.from_numpy(m).to(DEV), U.Scaling.FROBENIUS_GRAM)
    xo, to, _ = O.scale_and_orient(m, "gram")
    assert tall and to
    assert np.max(np.abs(x.cpu().numpy() - xo)) < 1e-14
    y = U.unso(x, U.default_coefficients())
    assert rel(y.cpu().numpy(), O.unso_poly(xo)) <= 1e-10
    y = U.muon_ns(x, 5)
    assert rel(y.cpu().numpy(), O.quintic_ns(xo, O.muon_rows(5))) <= 1e-10
    y = U.original_ns(x, 8)
    assert rel(y.cpu().numpy(), O.cubic_ns(xo, 8)) <= 1e-10


# ------------------------------------------------------------------ larger / BASELINE-shaped cases
@pytest.mark.parametrize("method", ["unso", "muon5"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_cfg2_full(precision, method):
    """configs[1]: 16 x 2048x512 controlled spectrum s ~ logU[1e-4, 1] against the oracle on the same
    (mode-rounded) input, UNSO and the Muon-5 comparison path: fp32 <= 1e-5, bf16 <= 2e-2."""
    rng = np.random.default_rng(2)
    ms = np.stack([O.controlled_spectrum_matrix(2048, 512, np.exp(rng.uniform(np.log(1e-4), 0, 512)), 100 + i)
                   for i in range(16)]).astype(np.float32)
    spec = (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()) if method == "unso"
            else U.MethodSpec(U.MethodKind.MUON_NS, iterations=5))
    res = U.orthogonalize(torch.from_numpy(ms).to(DEV), spec, precision=precision)
    y = res.y.double().cpu().numpy()
    worst = 0.0
    for i in range(16):
        inp = ms[i].astype(np.float64) if precision == "fp32" else bf16_round(ms[i])
        ref = O.run(inp, "unso")["y"] if method == "unso" else O.run(inp, "muon", iterations=5)["y"]
        worst = max(worst, rel(y[i], ref))
    print(f"cfg2 {method} {precision} worst rel err {worst:.2e}")
    assert worst <= TOL[precision]


@pytest.mark.parametrize("method", ["unso", "muon5"])
def test_cfg2_singular_value_map(method):
    """configs[1]'s stated purpose: the singular values of Y are the scalar map applied to the
    (scaled) singular values of X, g^N(s) (`scalar_map` ortho.py:286-310).  Y's spectrum is taken
    in fp64 on the device; the expected map is evaluated from the fp64 spectrum of the same
    (mode-rounded) input.  fp32 mode: |d sigma| <= 1e-5; bf16 mode: <= 2e-2."""
    rng = np.random.default_rng(2)
    ms = np.stack([O.controlled_spectrum_matrix(2048, 512, np.exp(rng.uniform(np.log(1e-4), 0, 512)), 100 + i)
                   for i in range(16)]).astype(np.float32)
    spec = (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()) if method == "unso"
            else U.MethodSpec(U.MethodKind.MUON_NS, iterations=5))
    fmap = U.scalar_map(spec)
    for precision, dtype in (("fp32", torch.float32), ("bf16", torch.bfloat16)):
        x = torch.from_numpy(ms).to(DEV, dtype)
        res = U.orthogonalize(x, spec, precision=precision)
        sy = torch.linalg.svdvals(res.y.double()).cpu().numpy()
        sx = torch.linalg.svdvals(x.double()).cpu().numpy()
        if method == "unso":   # gram scaling: X / ||X^T X||_F^(1/2)
            scale = (sx ** 4).sum(axis=1, keepdims=True) ** 0.25
        else:                  # plain scaling: X / ||X||_F
            scale = np.sqrt((sx ** 2).sum(axis=1, keepdims=True))
        want = np.sort(fmap(sx / scale), axis=1)[:, ::-1]
        got = np.sort(sy, axis=1)[:, ::-1]
        err = float(np.abs(got - want).max())
        print(f"cfg2 {method} {precision}: max |sigma(Y) - g(sigma(X))| = {err:.2e} "
              f"(sigma(Y) in [{got.min():.3e}, {got.max():.3e}])")
        assert err <= TOL[precision], (precision, err)


@pytest.mark.parametrize("shape,scale,seed", [((4096, 1024), 1.0, 5), ((1024, 1024), 0.02, 6), ((640, 1536), 1.0, 7)])
def test_bf16_mode_gaussian_shapes(shape, scale, seed):
    m = (O.gaussian_matrix(*shape, seed) * scale).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    res, y = run(m, spec, torch.bfloat16, "bf16")
    ref = O.run(bf16_round(m), "unso")["y"]
    r = rel(y, ref)
    print(f"bf16 {shape}: rel {r:.2e}")
    assert r <= TOL["bf16"]


def test_pareto_spectrum_both_modes():
    """configs[4]-like (reduced): heavy-tailed spectrum in [1e-6, 1], fp32 and bf16 modes."""
    rng = np.random.default_rng(4)
    s = 1.0 + rng.pareto(1.5, 512)
    s = 1e-6 + (s - s.min()) / (s.max() - s.min()) * (1.0 - 1e-6)
    m = O.controlled_spectrum_matrix(1536, 512, s, 44).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    _, y = run(m, spec, torch.float32, "fp32")
    r32 = rel(y, O.run(m.astype(np.float64), "unso")["y"])
    _, yb = run(m, spec, torch.float32, "bf16")
    rb = rel(yb, O.run(bf16_round(m), "unso")["y"])
    print(f"pareto: fp32 {r32:.2e}  bf16 {rb:.2e}")
    assert r32 <= TOL["fp32"]
    assert rb <= TOL["bf16"]


# ------------------------------------------------------------------ engine coverage (tcgen05 paths)
@pytest.mark.parametrize("shape", [(65536, 512), (512, 65536), (9000, 640), (640, 9000)])
def test_bf16_many_tiles_per_cta_pair(shape):
    """More work items than CTA pairs (multi-tile accumulator ring, phase tracking), tall and
    wide orientations, ragged h (640 is not a multiple of 256) -- against the oracle."""
    m = O.gaussian_matrix(*shape, 21).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    _, y = run(m, spec, torch.float32, "bf16")
    ref = O.run(bf16_round(m), "unso")["y"]
    r = rel(y, ref)
    print(f"bf16 {shape}: rel {r:.2e}")
    assert r <= TOL["bf16"]


def test_bf16_batched_persistent_chain():
    ms = np.stack([O.gaussian_matrix(1024, 256, 30 + i) for i in range(8)]).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    y = U.orthogonalize(torch.from_numpy(ms).to(DEV), spec, precision="bf16").y.double().cpu().numpy()
    for i in range(8):
        assert rel(y[i], O.run(bf16_round(ms[i]), "unso")["y"]) <= TOL["bf16"]


def test_bf16_multi_launch_chain_large_h():
    """h = 2304: 171 upper 128-tiles > 148 SMs -> the multi-launch chain path; ragged vs 256."""
    m = O.gaussian_matrix(4608, 2304, 40).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    _, y = run(m, spec, torch.float32, "bf16")
    r = rel(y, O.run(bf16_round(m), "unso")["y"])
    print(f"bf16 multi-launch chain h=2304: rel {r:.2e}")
    assert r <= TOL["bf16"]


def test_single_term_apply_option():
    m = O.gaussian_matrix(8192, 512, 41).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), apply_terms=1)
    _, y = run(m, spec, torch.float32, "bf16")
    r = rel(y, O.run(bf16_round(m), "unso")["y"])
    print(f"single-term apply: rel {r:.2e}")
    assert r <= TOL["bf16"]


@pytest.mark.slow
def test_cfg4_full_size_rows_against_oracle():
    """configs[3] at full size (262144 x 2048 bf16): 2048 sampled rows of Y against the
    oracle (fp64 Gram, chain and apply on the host), plus the whole Y against the
    fp32-mode (fp64-grade) device path on the same input."""
    g = torch.Generator(device=DEV).manual_seed(1234)
    x = torch.randn(262144, 2048, generator=g, device=DEV).to(torch.bfloat16)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    yb = U.orthogonalize(x, spec, precision="bf16").y
    y64 = U.orthogonalize(x.double(), spec, precision="fp32").y
    r_dev = float((yb.double() - y64).norm() / y64.norm())
    rows = np.sort(np.random.default_rng(0).choice(262144, 2048, replace=False))
    ref = O.unso_rows_of_tall(x.double().cpu().numpy(), rows)
    r_bf = rel(yb[torch.from_numpy(rows).to(DEV)].double().cpu().numpy(), ref)
    r_64 = rel(y64[torch.from_numpy(rows).to(DEV)].cpu().numpy(), ref)
    print(f"cfg4: bf16 vs oracle rows {r_bf:.2e}; fp32-mode vs oracle rows {r_64:.2e}; bf16 vs fp32-mode {r_dev:.2e}")
    assert r_64 <= 1e-6  # fp32 mode on the int8 digit engine: ~1e-7 (fp64 DMMA engine: ~1e-14)
    assert r_bf <= TOL["bf16"]
    assert r_dev <= TOL["bf16"]


def test_adaptive_apply_decision():
    """Default bf16 apply: P_lo is dropped on the device only when the bound allows it;
    a well-conditioned Gaussian takes the single-term path, an ill-conditioned one keeps two
    terms, and both stay within tolerance (and match the forced two-term path closely)."""
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    spec2 = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), apply_terms=2)
    g = O.gaussian_matrix(32768, 512, 50).astype(np.float32)
    rng = np.random.default_rng(51)
    s = np.exp(rng.uniform(np.log(1e-4), 0, 512))
    ill = O.controlled_spectrum_matrix(2048, 512, s, 52).astype(np.float32)
    for m, expect_single in ((g, True), (ill, False)):
        x = torch.from_numpy(m).to(DEV)
        res = U.orthogonalize(x, spec, precision="bf16")
        info = res.info[0]
        y = res.y.double().cpu().numpy()
        ref = O.run(bf16_round(m), "unso")["y"]
        r = rel(y, ref)
        r2 = rel(U.orthogonalize(x, spec2, precision="bf16").y.double().cpu().numpy(), ref)
        print(f"adaptive apply: single={info['apply_single']} bound={info['apply_bound']:.2e} rel={r:.2e} (two-term {r2:.2e})")
        assert bool(info["apply_single"]) == expect_single
        assert r <= TOL["bf16"]
        if expect_single:
            assert r <= info["apply_bound"] + 2 * r2


# ------------------------------------------------------------------ NS / Muon comparison path in bf16 mode
@pytest.mark.parametrize("name", ["muon5", "muon3", "original4", "cesista", "external"])
def test_ns_bf16_mode_small_cases(golden_arrays, golden_kats, name):
    for key in ("in_64x256", "in_130x66", "in_16x40", "in_40x16"):
        m = golden_arrays[key].astype(np.float32)
        _, y = run(m, spec_for(name, golden_kats), torch.float32, "bf16")
        ref = O.run(bf16_round(m), **oracle_kw(name, golden_kats))["y"]
        r = rel(y, ref)
        assert r <= TOL["bf16"], (name, key, r)


def test_ns_bf16_cfg1_and_large():
    g = O.gaussian_matrix(512, 128, 0).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)
    _, y = run(g, spec, torch.float32, "bf16")
    r = rel(y, O.run(bf16_round(g), "muon", iterations=5)["y"])
    print(f"cfg1 muon5 bf16: rel {r:.2e}")
    assert r <= TOL["bf16"]
    m = (O.gaussian_matrix(3000, 1024, 61) * 0.02).astype(np.float32)   # cfg3-like, ragged w
    _, y = run(m, spec, torch.float32, "bf16")
    r = rel(y, O.run(bf16_round(m), "muon", iterations=5)["y"])
    print(f"3000x1024 muon5 bf16: rel {r:.2e}")
    assert r <= TOL["bf16"]
    ms = np.stack([O.gaussian_matrix(256, 768, 70 + i) for i in range(3)]).astype(np.float32)
    yb = U.orthogonalize(torch.from_numpy(ms).to(DEV), spec, precision="bf16").y.double().cpu().numpy()
    for i in range(3):
        assert rel(yb[i], O.run(bf16_round(ms[i]), "muon", iterations=5)["y"]) <= TOL["bf16"]


def test_bf16_glue_free_route_ragged_batch():
    """Batch whose tiles exceed co-residency and fill >= 2 waves: K1 writes G as bf16 hi/lo +
    norm partials directly (no split-K), the first squaring folds C_1 = G/s^2, the last emits
    P statistics; ragged h (640) and w (900)."""
    ms = np.stack([O.gaussian_matrix(900, 640, 80 + i) for i in range(48)]).astype(np.float32)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    res = U.orthogonalize(torch.from_numpy(ms).to(DEV), spec, precision="bf16")
    y = res.y.double().cpu().numpy()
    worst = max(rel(y[i], O.run(bf16_round(ms[i]), "unso")["y"]) for i in range(0, 48, 6))
    print(f"glue-free ragged batch: worst rel {worst:.2e}; apply_single={res.info[0]['apply_single']}")
    assert worst <= TOL["bf16"]


@pytest.mark.parametrize("kind", ["cfg3-square", "cfg3-tall", "cfg2-spectrum", "cfg5-pareto"])
def test_chain_fp8_cross_terms_vs_bf16x3(kind):
    """Large-h chain recipes (glue-free route, h = 2304 > co-residency): default hi*hi (bf16) +
    e4m3 cross terms vs the bf16x3 chain, both against the oracle on the same rounded input."""
    rng = np.random.default_rng(90)
    if kind == "cfg3-square":
        m = O.gaussian_matrix(2304, 2304, 91) * 0.02
    elif kind == "cfg3-tall":
        m = O.gaussian_matrix(8064, 2304, 92) * 0.02
    elif kind == "cfg2-spectrum":
        m = O.controlled_spectrum_matrix(4608, 2304, np.exp(rng.uniform(np.log(1e-4), 0, 2304)), 93)
    else:
        s = 1 + rng.pareto(1.5, 2304)
        m = O.controlled_spectrum_matrix(4608, 2304, 1e-6 + (s - s.min()) / (s.max() - s.min()) * (1 - 1e-6), 94)
    m = m.astype(np.float32)
    ref = O.run(bf16_round(m), "unso")["y"]
    out = {}
    for chain in (None, "bf16x3"):
        spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), chain=chain)
        _, y = run(m, spec, torch.float32, "bf16")
        out[chain or "bf16+e4m3"] = rel(y, ref)
    print(f"chain recipes {kind}: {out}")
    assert all(v <= TOL["bf16"] for v in out.values())
    assert out["bf16+e4m3"] <= 1e-2


def test_graphed_orthogonalize_matches_eager():
    from paper_2602_02500_b200.graphs import GraphedOrthogonalize
    g0 = O.gaussian_matrix(512, 128, 0).astype(np.float32)
    g1 = O.gaussian_matrix(512, 128, 1).astype(np.float32)
    for prec, spec in (("fp32", U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())),
                       ("bf16", U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())),
                       ("fp32", U.MethodSpec(U.MethodKind.MUON_NS, iterations=5))):
        x0 = torch.from_numpy(g0).to(DEV)
        x1 = torch.from_numpy(g1).to(DEV)
        gr = GraphedOrthogonalize(x0, spec, precision=prec)
        for x in (x1, x0):
            y = gr(x).clone()
            e = U.orthogonalize(x, spec, precision=prec).y
            assert torch.equal(y, e), prec
    ms = np.stack([O.gaussian_matrix(2048, 512, 200 + i) for i in range(16)]).astype(np.float32)
    xb = torch.from_numpy(ms).to(DEV)
    gr = GraphedOrthogonalize(xb, U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()), precision="bf16")
    assert torch.equal(gr(xb).clone(), U.orthogonalize(xb, gr.spec, precision="bf16").y)


def test_chain_truncation_well_conditioned():
    """Tall Gaussian (kappa ~ 1.2): the persistent chain stops early and the result
    stays within the bf16 tolerance of the oracle and within the truncation bound of the full chain."""
    g = torch.Generator().manual_seed(12)
    x = torch.randn(65536, 512, generator=g).to(torch.bfloat16).to(DEV)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    res = U.orthogonalize(x, spec, precision="bf16")
    full = U.orthogonalize(x, U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), truncate=False),
                           precision="bf16")
    torch.cuda.synchronize()
    steps, steps_full = res.info[0]["chain_steps"], full.info[0]["chain_steps"]
    print(f"chain steps: {steps} (full {steps_full})")
    assert steps_full == 13 and 0 < steps < 13
    rows = np.arange(4096)  # row sample of the oracle (the same P applies to every row)
    ref = O.unso_rows_of_tall(x.double().cpu().numpy(), rows)
    y = res.y.double().cpu().numpy()
    yf = full.y.double().cpu().numpy()
    d = rel(y, yf)
    r = rel(y[rows], ref)
    print(f"truncated vs full chain: {d:.2e}; vs oracle rows: {r:.2e}")
    assert d <= 2.0 ** -12 + 2.0 ** -9  # truncation bound + bf16 output rounding
    assert r <= TOL["bf16"]


def test_chain_truncation_not_taken_when_ill_conditioned():
    g = torch.Generator().manual_seed(13)
    x = torch.randn(512, 512, generator=g).to(torch.bfloat16).to(DEV)
    res = U.orthogonalize(x, U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()), precision="bf16")
    torch.cuda.synchronize()
    assert res.info[0]["chain_steps"] == 13
    ref = O.run(x.double().cpu().numpy(), "unso")["y"]
    assert rel(res.y.double().cpu().numpy(), ref) <= TOL["bf16"]


@pytest.mark.parametrize("precision,h", [("bf16", 512), ("bf16", 2048), ("fp32", 256)])
def test_row_sharded_native_stages_match_unsharded(precision, h):
    """The cfg4 scheme on one GPU: per-shard Gram (unso_gram), the sum of the shard Grams standing in for
    the NCCL all-reduce, then unso_orthogonalize_from_gram per shard; the concatenated rows equal the
    unsharded orthogonalize and the oracle (row sample)."""
    from paper_2602_02500_b200.distributed import native_finish, native_gram, row_shard_bounds
    g = torch.Generator().manual_seed(14 + h)
    w = 16 * h
    x = torch.randn(w, h, generator=g).to(torch.bfloat16 if precision == "bf16" else torch.float32).to(DEV)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    world = 4
    shards = [x[slice(*row_shard_bounds(w, world, r))] for r in range(world)]
    gsum = sum(native_gram(s, spec, precision) for s in shards)
    ys = [native_finish(s, gsum.clone(), spec, precision)[0] for s in shards]
    y = torch.cat(ys)
    full = U.orthogonalize(x, spec, precision=precision).y
    torch.cuda.synchronize()
    rows = np.arange(0, w, 7)[:2048]
    ref = O.unso_rows_of_tall(x.double().cpu().numpy(), rows)
    tol = TOL[precision] + (2.0 ** -9 if precision == "bf16" else 0.0)
    assert rel(y.double().cpu().numpy()[rows], ref) <= tol
    assert rel(y.double().cpu().numpy(), full.double().cpu().numpy()) <= (5e-3 if precision == "bf16" else 1e-6)


@pytest.mark.parametrize("h", [128, 256])
def test_fp32_persistent_chain_truncation(h):
    """fp32 mode, h <= 256: one cooperative launch runs the fp64 chain; a well-conditioned input
    stops early (dropped terms <= 2^-30 relative) and stays within 1e-5 of the oracle."""
    g = torch.Generator().manual_seed(40 + h)
    x = torch.randn(64 * h, h, generator=g, dtype=torch.float64).float().to(DEV)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    res = U.orthogonalize(x, spec, precision="fp32")
    full = U.orthogonalize(x, U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), truncate=False),
                           precision="fp32")
    torch.cuda.synchronize()
    steps = res.info[0]["chain_steps"]
    print(f"h={h}: fp64 chain steps {steps} (full {full.info[0]['chain_steps']})")
    assert 0 < steps < 13 and full.info[0]["chain_steps"] == 13
    rows = np.arange(0, 64 * h, 5)
    ref = O.unso_rows_of_tall(x.double().cpu().numpy(), rows)
    assert rel(res.y.double().cpu().numpy()[rows], ref) <= TOL["fp32"]
    assert rel(res.y.double().cpu().numpy(), full.y.double().cpu().numpy()) <= 1e-7


@pytest.mark.parametrize("h,world", [(512, 4), (2048, 4), (640, 3)])
def test_nvlink_gram_reduction_emulated_ranks(h, world):
    """The peer-memory Gram reduction (unso_gram_push / _reduce / _wait) with `world`
    ranks emulated on one GPU phase by phase: every rank ends with the same bit-identical reduced
    Gram, equal to the sum of the shard Grams, and the sharded orthogonalization matches the
    unsharded one."""
    from paper_2602_02500_b200.distributed import (NvlinkGramReducer, gram_push_splits, native_finish, native_gram,
                                                   row_shard_bounds)
    g = torch.Generator().manual_seed(50 + h)
    w = 8 * h
    x = torch.randn(w, h, generator=g).to(torch.bfloat16).to(DEV)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    shards = [x[slice(*row_shard_bounds(w, world, r))] for r in range(world)]
    splits = gram_push_splits(h, min(s.shape[0] for s in shards))
    reducers = NvlinkGramReducer.emulated(h, world, splits, DEV)
    for it in range(2):  # two calls: the epoch-tagged flags need no reset
        for r in range(world):
            reducers[r].push(shards[r], spec, "bf16")
        for r in range(world):
            reducers[r].reduce()
        gs = [reducers[r].wait() for r in range(world)]
        torch.cuda.synchronize()
        for r in range(1, world):
            assert torch.equal(gs[r], gs[0])
        ref = sum(native_gram(s, spec, "bf16").double() for s in shards)
        assert float((gs[0].double() - ref).norm() / ref.norm()) <= 1e-6
    y = torch.cat([native_finish(s, gs[r].clone(), spec, "bf16")[0] for r, s in enumerate(shards)])
    full = U.orthogonalize(x, spec, precision="bf16").y
    torch.cuda.synchronize()
    # against the oracle (ortho.py:140-205 on the same bf16 values), on rows of every rank's shard
    rows = np.arange(0, w, 3)
    ref = O.unso_rows_of_tall(x.double().cpu().numpy(), rows)
    r_or = rel(y.double().cpu().numpy()[rows], ref)
    print(f"nvlink-reduced h={h} world={world}: vs oracle rows {r_or:.2e}")
    assert r_or <= TOL["bf16"] + 2.0 ** -9
    assert rel(y.double().cpu().numpy(), full.double().cpu().numpy()) <= 5e-3


def test_nvlink_gram_reduction_symmetric_memory_world1():
    """The same path through torch symmetric memory (the real peer mappings) on a 1-rank group."""
    import os
    import torch.distributed as dist
    from paper_2602_02500_b200.distributed import orthogonalize_row_sharded
    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        g = torch.Generator().manual_seed(77)
        x = torch.randn(16384, 1024, generator=g).to(torch.bfloat16).to(DEV)
        spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
        try:
            y = orthogonalize_row_sharded(x, spec, collective="nvlink")
        except (RuntimeError, NotImplementedError) as exc:  # symmetric memory unavailable on this node
            pytest.skip(f"torch symmetric memory unavailable: {exc}")
        full = U.orthogonalize(x, spec).y
        torch.cuda.synchronize()
        assert rel(y.double().cpu().numpy(), full.double().cpu().numpy()) <= 5e-3
    finally:
        if own:
            from paper_2602_02500_b200 import distributed as D
            D._REDUCERS.clear()
            dist.destroy_process_group()
