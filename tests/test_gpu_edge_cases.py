"""GPU edge cases of the drop-in boundary, each checked against the CPU oracle on the same values
(tolerances as in test_gpu_parity.py: fp32 mode 1e-5, bf16 mode 2e-2 on the bf16-rounded input).

Covers what the reference's own tests exercise around the kernels (tests/test_ortho.py shapes,
degenerate inputs, orientation) plus the layouts a torch caller hands over: strided rows whose
leading dimension breaks TMA's 16-byte rule, transposed views, strided batches, tiny and odd shapes,
h just past a tile edge, square inputs, fp64 I/O, out=, and a zero matrix inside a batch."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
TOL = {"fp32": 1e-5, "bf16": 2e-2}
UNSO = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
MUON = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def oracle_of(x: torch.Tensor, method: str, precision: str) -> np.ndarray:
    """Oracle output for the values the kernel actually sees (bf16-rounded in bf16 mode)."""
    v = x.detach().to(torch.bfloat16 if precision == "bf16" else x.dtype).double().cpu().numpy()
    kw = {"iterations": 5} if method == "muon" else {}
    if v.ndim == 2:
        return O.run(v, method, **kw)["y"]
    return np.stack([O.run(m, method, **kw)["y"] for m in v])


def check(x, spec, method, precision, **kw):
    res = U.orthogonalize(x, spec, precision=precision, **kw)
    torch.cuda.synchronize()
    assert res.y.shape == x.shape and res.y.dtype == x.dtype
    r = rel(res.y.double().cpu().numpy(), oracle_of(x, method, precision))
    # a bf16 OUTPUT carries its own rounding: round-to-nearest bounds it by 2^-9 relative (Frobenius)
    tol = TOL[precision] + (2.0 ** -9 if x.dtype == torch.bfloat16 else 0.0)
    assert r <= tol, (tuple(x.shape), precision, method, r)
    return res


def gaussian(shape, seed, dtype=torch.float32):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(*shape, generator=g, dtype=torch.float64).to(dtype).to(DEV)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (2, 3), (3, 2), (5, 5), (8, 8), (9, 17)])
def test_tiny_shapes(shape, precision):
    x = gaussian(shape, 11 + shape[0] * 31 + shape[1])
    check(x, UNSO, "unso", precision)
    if precision == "fp32":
        check(x, MUON, "muon", precision)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(300, 37), (37, 1000), (129, 700), (700, 129), (257, 1200), (1300, 255),
                                   (384, 384), (1000, 1000)])
def test_odd_and_tile_edge_shapes(shape, precision):
    """h not a multiple of 8, h one past a 128 / 256 tile, square inputs (not transposed)."""
    x = gaussian(shape, 100 + shape[0] + shape[1])
    res = check(x, UNSO, "unso", precision)
    assert res.was_transposed == (shape[0] > shape[1])


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_strided_rows_unaligned_ld(precision, dtype):
    """Row stride (ld) = cols + 5: not a multiple of 8 elements, so TMA cannot read it in place."""
    for rows, cols in ((600, 200), (200, 600)):
        big = gaussian((rows, cols + 5), rows + cols, dtype)
        x = big[:, :cols]
        assert x.stride(0) == cols + 5
        res = check(x, UNSO, "unso", precision)
        ref = U.orthogonalize(x.contiguous(), UNSO, precision=precision).y
        assert torch.equal(res.y, ref)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_transposed_view_and_strided_batch(precision):
    base = gaussian((6, 300, 120), 5)
    xt = base[0].t()                      # (120, 300) view with stride(-1) != 1
    check(xt, UNSO, "unso", precision)
    xb = base[::2]                        # batch stride 2 x 300 x 120
    res = check(xb, UNSO, "unso", precision)
    single = torch.stack([U.orthogonalize(m.contiguous(), UNSO, precision=precision).y for m in xb])
    assert rel(res.y.double().cpu().numpy(), single.double().cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_batches_of_wide_and_tall(precision):
    check(gaussian((3, 96, 400), 21), UNSO, "unso", precision)
    check(gaussian((3, 400, 96), 22), UNSO, "unso", precision)


def test_many_tiny_matrices():
    x = gaussian((512, 16, 8), 33)
    for precision in ("fp32", "bf16"):
        check(x, UNSO, "unso", precision)
    check(x, MUON, "muon", "fp32")


def test_fp64_io_both_precisions():
    x = gaussian((500, 140), 44, torch.float64)
    res = U.orthogonalize(x, UNSO, precision="fp32")
    assert res.y.dtype == torch.float64
    assert rel(res.y.cpu().numpy(), O.run(x.cpu().numpy(), "unso")["y"]) <= 1e-10
    check(x, UNSO, "unso", "bf16")


def test_out_parameter_and_input_untouched():
    x = gaussian((4, 256, 64), 55)
    keep = x.clone()
    out = torch.empty_like(x)
    res = U.orthogonalize(x, UNSO, precision="bf16", out=out)
    assert res.y.data_ptr() == out.data_ptr()
    assert torch.equal(x, keep)
    with pytest.raises(U.ShapeError):
        U.orthogonalize(x, UNSO, out=torch.empty(4, 64, 256, device=DEV))


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_zero_matrix_inside_batch_is_degenerate(precision):
    x = gaussian((3, 200, 50), 66)
    x[1].zero_()
    with pytest.raises(U.DegenerateInputError):
        U.orthogonalize(x, UNSO, precision=precision)
    # the other matrices are still computed (status is per matrix)
    res = U.orthogonalize(x, UNSO, precision=precision, check=False)
    torch.cuda.synchronize()
    for i in (0, 2):
        assert rel(res.y[i].double().cpu().numpy(), oracle_of(x[i], "unso", precision)) <= TOL[precision]


def test_scale_invariance():
    """Both scalings are scale-invariant (ortho.py:153-165): Y(c X) == Y(X) up to rounding."""
    x = gaussian((400, 100), 77, torch.float64)
    a = U.orthogonalize(x, UNSO, precision="fp32").y
    b = U.orthogonalize(x * 1e3, UNSO, precision="fp32").y
    assert rel(b.cpu().numpy(), a.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
def test_ns_layouts_vectorized_and_fallback(precision, dtype):
    """The NS comparison path (plain-scaling norm + state initialisation) on layouts that take the
    16-byte-chunk kernels (contiguous, cols % 8 == 0) and ones that fall back to the element kernels
    (cols % 8 != 0, unaligned row stride), tall and wide, single and batched."""
    cases = [gaussian((640, 96), 61, dtype), gaussian((96, 640), 62, dtype), gaussian((3, 300, 52), 63, dtype),
             gaussian((250, 37), 64, dtype), gaussian((400, 133), 65, dtype)[:, :130]]
    for x in cases:
        check(x, MUON, "muon", precision)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float64])
def test_method_mode_dtype_matrix(mode, dtype):
    """Every method kind and scaling x precision mode x input dtype, tall and wide, on an
    ill-conditioned (log-uniform, 1e-4) spectrum, against the oracle on the values the mode computes
    on (profiles/round1_parity_sweep_methods_modes_dtypes.txt has the wider sweep)."""
    ces = U.CesistaStepParams(U.default_cesista_triples())
    methods = [
        (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()), dict(method="unso")),
        (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="plain"),
         dict(method="unso", scaling="plain")),
        (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="gelfand"),
         dict(method="unso", scaling="gelfand")),
        (MUON, dict(method="muon", iterations=5)),
        (U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=8), dict(method="original", iterations=8)),
        (U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=ces),
         dict(method="cesista", rows=O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES))),
    ]
    rng = np.random.default_rng(3)
    for shape in ((1024, 256), (256, 1024)):
        m = O.controlled_spectrum_matrix(*shape, np.exp(rng.uniform(np.log(1e-4), 0.0, 256)), 70 + shape[0])
        x = torch.from_numpy(m).to(DEV, dtype)
        vals = (x if mode == "fp32" else x.to(torch.bfloat16)).double().cpu().numpy()
        tol = TOL[mode] + (2.0 ** -9 if dtype == torch.bfloat16 else 0.0)
        for spec, kw in methods:
            y = U.orthogonalize(x, spec, precision=mode).y
            assert y.dtype == dtype
            r = rel(y.double().cpu().numpy(), O.run(vals, **kw)["y"])
            assert r <= tol, (shape, mode, dtype, kw, r)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_ns_batched_tall_and_wide(precision):
    """Batched NS (Muon-5, cubic) calls equal the oracle per matrix, tall and wide, with a matrix of a
    different scale in the batch (per-matrix plain scaling)."""
    for shape in ((4, 600, 200), (4, 200, 600)):
        x = gaussian(shape, 90 + shape[1])
        x[2] *= 1e-3
        check(x, MUON, "muon", precision)
        orig = U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=6)
        res = U.orthogonalize(x, orig, precision=precision)
        vals = (x if precision == "fp32" else x.to(torch.bfloat16)).double().cpu().numpy()
        ref = np.stack([O.run(m, "original", iterations=6)["y"] for m in vals])
        assert rel(res.y.double().cpu().numpy(), ref) <= TOL[precision]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("power", [1, 3])
def test_gelfand_powers(precision, power):
    """Gelfand scaling ||(A A^T)^k||_F^(1/(2k)) for k != 2 (ortho.py:158-163), UNSO and Muon-5."""
    x = gaussian((700, 180), 120 + power)
    vals = (x if precision == "fp32" else x.to(torch.bfloat16)).double().cpu().numpy()
    for spec, kw in ((U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling="gelfand",
                                   gelfand_power=power), dict(method="unso")),
                     (U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, scaling="gelfand", gelfand_power=power),
                      dict(method="muon", iterations=5))):
        y = U.orthogonalize(x, spec, precision=precision).y.double().cpu().numpy()
        ref = O.run(vals, scaling="gelfand", gelfand_power=power, **kw)["y"]
        assert rel(y, ref) <= TOL[precision], (power, precision, kw, rel(y, ref))


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("order,rule", [(2, "exact"), (6, "approx-sum"), (20, "approx-abs"), (20, "exact")])
def test_other_polynomial_orders_and_rules(precision, order, rule):
    """CoefficientSets of other orders N and b-rules (scalarpoly.py:39-61, 117-127) on the small
    (h <= 128), persistent (h <= 2048) and multi-launch routes, against the oracle."""
    rng = np.random.default_rng(order)
    a = rng.uniform(-1.0, 2.0, order - 1)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.CoefficientSet(order, a, rule))
    for shape in ((600, 96), (1200, 384)):
        x = gaussian(shape, 130 + order + shape[1])
        vals = (x if precision == "fp32" else x.to(torch.bfloat16)).double().cpu().numpy()
        y = U.orthogonalize(x, spec, precision=precision).y.double().cpu().numpy()
        ref = O.run(vals, "unso", order=order, a=a, rule=rule)["y"]
        assert rel(y, ref) <= TOL[precision], (order, rule, shape, precision, rel(y, ref))


def test_other_order_on_the_multi_launch_route():
    """h = 2304 (> the persistent chain's co-residency): the CTA-pair squaring launches with N = 8."""
    rng = np.random.default_rng(8)
    a = rng.uniform(-1.0, 2.0, 7)
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.CoefficientSet(8, a, "exact"))
    x = gaussian((4608, 2304), 140)
    y = U.orthogonalize(x, spec, precision="bf16").y.double().cpu().numpy()
    ref = O.run(x.to(torch.bfloat16).double().cpu().numpy(), "unso", order=8, a=a, rule="exact")["y"]
    assert rel(y, ref) <= TOL["bf16"], rel(y, ref)


def test_extreme_scales():
    """fp32 mode (fp64 accumulation) handles the input's full range like the reference; bf16 mode
    accumulates the Gram in fp32, so inputs whose Gram leaves the fp32 range are reported loudly as
    degenerate instead of returning garbage."""
    x = gaussian((400, 100), 150, torch.float32)
    base = U.orthogonalize(x, UNSO, precision="fp32").y
    for c in (1e-25, 1e18):
        y = U.orthogonalize(x * c, UNSO, precision="fp32").y
        assert rel(y.double().cpu().numpy(), base.double().cpu().numpy()) <= 1e-6, c
        with pytest.raises(U.DegenerateInputError):
            U.orthogonalize(x * c, UNSO, precision="bf16")


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_non_finite_input_is_degenerate(precision, bad):
    """A NaN / Inf entry makes the scaling denominator non-finite: DegenerateInputError, as the
    reference's preprocess raises (ortho.py:164-165), for UNSO and the NS kinds."""
    x = gaussian((300, 80), 160)
    x[5, 7] = bad
    for spec in (UNSO, MUON):
        with pytest.raises(U.DegenerateInputError):
            U.orthogonalize(x, spec, precision=precision)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_wide_large_h(precision):
    """Wide input (rows < cols) with h = 2304 > the persistent chain's co-residency: the multi-launch
    chain and the MN-major apply, UNSO and Muon-5 (hi/lo state on the wide path)."""
    x = gaussian((2304, 4608), 170)
    check(x, UNSO, "unso", precision)
    check(x, MUON, "muon", precision)


def test_side_streams_run_concurrently_and_match():
    """Calls on two side streams at once (per-stream workspaces, stream-ordered ABI) equal the
    default-stream results bit for bit."""
    xa = gaussian((4, 1024, 256), 180, torch.bfloat16)
    xb = gaussian((2048, 512), 181)
    ref_a = U.orthogonalize(xa, UNSO).y
    ref_b = U.orthogonalize(xb, MUON, precision="bf16").y
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            ya = U.orthogonalize(xa, UNSO, check=False).y
        with torch.cuda.stream(s2):
            yb = U.orthogonalize(xb, MUON, precision="bf16", check=False).y
        outs.append((ya, yb))
    torch.cuda.synchronize()
    for ya, yb in outs:
        assert torch.equal(ya, ref_a)
        assert torch.equal(yb, ref_b)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_two_step_api_on_bf16_input(precision):
    """unso(preprocess(x)) on a bf16 tall input: preprocess returns the rescaled, transposed copy in
    fp32 (the reference keeps it in fp64, ortho.py:167), not a second bf16 rounding, so the fp32
    mode reaches 1e-5 of the oracle on the bf16 values and the bf16 mode stays within its bar."""
    x = gaussian((1000, 300), 77).to(torch.bfloat16)
    xs, tall = U.preprocess(x, U.Scaling.FROBENIUS_GRAM)
    assert tall and xs.dtype == torch.float32 and xs.shape == (300, 1000)
    y = U.unso(xs, U.default_coefficients(), precision=precision)
    ref = O.run(x.double().cpu().numpy(), "unso")["y"].T
    r = rel(y.double().cpu().numpy(), ref)
    assert r <= TOL[precision], (precision, r)
