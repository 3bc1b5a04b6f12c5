"""Element-wise full-size parity at BASELINE configs[2] and configs[4]: long-side samples of Y
(rows of a tall result, columns of a wide or square one) against the CPU oracle on the same input
values (oracle.unso_sampled / quintic_sampled: the reference's Gram, scale, squaring chain and
polynomial in fp64, ortho.py:140-205 and :221-231, with P applied only to the sampled columns).

Unlike the spectral check of test_gpu_fullsize.py, this sees the singular VECTORS: a Y with the
right spectrum but wrong vectors fails here.  Bars: relative Frobenius error of the sampled block
<= 2e-2 in bf16 mode (+ 2^-9 for a bf16 output) and <= 1e-5 in fp32 mode.

Host cost: the oracle's 13 fp64 squarings of the h x h B are ~1.8 TFLOP at h = 4096 and ~14 TFLOP
at h = 8192 (OpenBLAS on the box's host cores); the configs[4] oracle is computed once and shared by
both modes (its input holds bf16-representable values, so both modes see the same numbers)."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
TOL = {"fp32": 1e-5, "bf16": 2e-2}
SAMPLES = 256


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def sampled(y: torch.Tensor, idx: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(idx).to(DEV)
    tall = y.shape[0] > y.shape[1]
    return (y[t] if tall else y[:, t]).double().cpu().numpy()


def gaussian_bf16(rows, cols, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return (torch.randn(rows, cols, generator=g, device=DEV) * 0.02).to(torch.bfloat16)


UNSO = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
MUON = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)


@pytest.mark.parametrize("shape", [(4096, 4096), (14336, 4096), (4096, 14336)])
@pytest.mark.parametrize("method", ["unso", "muon5"])
def test_cfg3_shapes_sampled_against_oracle(shape, method):
    """configs[2]: q/k/v/o 4096^2 (square: not transposed, row Gram), up/gate 14336 x 4096 (tall),
    down 4096 x 14336 (wide), bf16, N(0, 0.02^2), bf16 mode."""
    x = gaussian_bf16(*shape, seed=700 + shape[0] + 3 * shape[1] + (1 if method == "muon5" else 0))
    spec = UNSO if method == "unso" else MUON
    y = U.orthogonalize(x, spec, precision="bf16").y
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    idx = np.sort(np.random.default_rng(shape[0] + shape[1]).choice(max(shape), SAMPLES, replace=False))
    m = x.double().cpu().numpy()
    ref = O.unso_sampled(m, idx) if method == "unso" else O.quintic_sampled(m, idx)
    r = rel(sampled(y, idx), ref)
    print(f"configs[2] {shape} {method} bf16: sampled rel err vs oracle {r:.2e}")
    assert r <= TOL["bf16"] + 2.0 ** -9, (shape, method, r)


@pytest.fixture(scope="module")
def cfg5_case():
    from test_gpu_fullsize import pareto_spectrum_matrix
    x = pareto_spectrum_matrix(16384, 8192, 4).to(torch.bfloat16).float()  # bf16-representable fp32 values
    idx = np.sort(np.random.default_rng(5).choice(16384, SAMPLES, replace=False))
    ref = O.unso_sampled(x.double().cpu().numpy(), idx)
    return x, idx, ref


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_cfg5_sampled_against_oracle(cfg5_case, precision):
    """configs[4]: 16384 x 8192 fp32 with a Pareto(1.5) spectrum in [1e-6, 1] (Haar U, V), both modes
    on the same values: bf16 mode (tcgen05 Gram, bf16 + e4m3 chain, bf16x2 apply) and fp32 mode
    (fp64-grade DMMA engine)."""
    x, idx, ref = cfg5_case
    y = U.orthogonalize(x, UNSO, precision=precision).y
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    r = rel(sampled(y, idx), ref)
    print(f"configs[4] 16384x8192 {precision}: sampled rel err vs oracle {r:.2e}")
    assert r <= TOL[precision], (precision, r)


def test_cfg5_batch_member_matches_single_call(cfg5_case):
    """The batched configs[4] call (here 2 matrices) gives each member the single-call result."""
    x, idx, ref = cfg5_case
    xb = torch.stack([x.flip(0), x])
    y = U.orthogonalize(xb, UNSO, precision="bf16").y
    torch.cuda.synchronize()
    r = rel(sampled(y[1], idx), ref)
    print(f"configs[4] batch member 1: sampled rel err vs oracle {r:.2e}")
    assert r <= TOL["bf16"]
