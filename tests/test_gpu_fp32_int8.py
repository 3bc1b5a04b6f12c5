"""fp32 mode on the int8 tensor cores (csrc/ozaki_i8.cuh): the Gram (ortho.py:156/198), the squarings
(ortho.py:201-203) and the apply (ortho.py:205) as exact int8 digit products (5 digits per operand,
15 tcgen05.mma kind::i8 products, fp64 combination) -- checked against the CPU oracle at the fp32-mode
bar (1e-5 relative Frobenius, BASELINE north_star) and against the fp64 DMMA engine
(`fp32_engine="dmma"`), plus the Gram alone against an fp64 product (split-K over K > 65536 included)."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def spec(**kw):
    return U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), **kw)


def controlled(rows, cols, lo, seed):
    rng = np.random.default_rng(seed)
    k = min(rows, cols)
    s = np.exp(rng.uniform(np.log(lo), 0.0, k))
    return O.controlled_spectrum_matrix(rows, cols, s, seed + 1)


CASES = [
    # (shape, kind, dtype, scaling)
    ((2048, 512), "logu", torch.float32, None),     # configs[1] matrix
    ((1000, 333), "gauss", torch.float32, None),    # tall, ragged h
    ((300, 700), "gauss", torch.float32, None),     # wide, ragged h
    ((640, 640), "logu", torch.float32, None),      # square
    ((900, 400), "gauss", torch.bfloat16, None),    # bf16 input
    ((700, 300), "gauss", torch.float64, None),     # fp64 input
    ((1200, 520), "logu", torch.float32, "plain"),
    ((1200, 520), "logu", torch.float32, "gelfand"),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_int8_engine_matches_oracle(case):
    shape, kind, dtype, scaling = CASES[case]
    m = controlled(*shape, 1e-4, 10 + case) if kind == "logu" else np.random.default_rng(case).standard_normal(shape)
    x = torch.from_numpy(m).to(dtype).to(DEV)
    res = U.orthogonalize(x, spec(scaling=scaling), precision="fp32")
    dm = U.orthogonalize(x, spec(scaling=scaling, fp32_engine="dmma"), precision="fp32")
    torch.cuda.synchronize()
    src = x.double().cpu().numpy()
    ref = O.run(src, "unso", scaling=scaling)["y"]
    y = res.y.double().cpu().numpy()
    e_or = rel(y, ref)
    e_dm = rel(y, dm.y.double().cpu().numpy())
    print(f"{shape} {kind} {str(dtype)[6:]} {scaling}: vs oracle {e_or:.2e}, vs fp64 DMMA {e_dm:.2e}")
    tol = 1e-5 + (2.0 ** -9 if dtype == torch.bfloat16 else 0.0)  # bf16 output rounding
    assert e_or <= tol
    assert e_dm <= (tol if dtype == torch.bfloat16 else 2e-6)


def test_int8_engine_batch_strided():
    """A batch of configs[1]-like matrices as a strided view (non-contiguous batch)."""
    ms = np.stack([controlled(1024, 384, 1e-4, 40 + i) for i in range(3)])
    big = torch.zeros(3, 1024, 400, dtype=torch.float32, device=DEV)
    big[:, :, :384] = torch.from_numpy(ms).float().to(DEV)
    x = big[:, :, :384]
    res = U.orthogonalize(x, spec(), precision="fp32")
    torch.cuda.synchronize()
    for b in range(3):
        ref = O.run(x[b].double().cpu().numpy(), "unso")["y"]
        assert rel(res.y[b].double().cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("rows,cols", [(4096, 640), (140000, 300)])
def test_int8_gram_against_fp64(rows, cols):
    """The Gram alone (unso_gram, fp32 mode) against the fp64 product: ~2^-41 relative per digit
    product, far below the fp32-mode bar; 140000 rows force split-K slices within the int32 bound."""
    from paper_2602_02500_b200.distributed import native_gram
    g = torch.Generator().manual_seed(rows)
    x = torch.randn(rows, cols, generator=g).to(DEV)
    G = native_gram(x, spec(), "fp32")
    torch.cuda.synchronize()
    xd = x.double()
    ref = (xd.T @ xd).cpu().numpy()
    err = rel(G.double().cpu().numpy(), ref)
    print(f"Gram {rows}x{cols}: {err:.2e}")
    assert err <= 1e-9


def test_int8_engine_poisoned_workspace():
    """Stale digit planes / maxima never leak into a later call (workspace pre-filled with 0xFF)."""
    x = torch.from_numpy(controlled(777, 555, 1e-4, 3)).float().to(DEV)
    buf = U.ortho.workspace_pool.get(512 << 20, DEV, torch.cuda.current_stream(DEV))
    buf.fill_(0xFF)
    torch.cuda.synchronize()
    y = U.orthogonalize(x, spec(), precision="fp32").y
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    ref = O.run(x.double().cpu().numpy(), "unso")["y"]
    assert rel(y.double().cpu().numpy(), ref) <= 1e-5


def test_int8_engine_nonfinite_input_is_flagged():
    """A NaN in the input must surface as a degenerate-input error (status word), not as a finite Y."""
    x = torch.randn(600, 400, device=DEV)
    x[17, 5] = float("nan")
    with pytest.raises(U.DegenerateInputError):
        U.orthogonalize(x, spec(), precision="fp32")


SWEEP = list(range(16))


@pytest.mark.parametrize("case", SWEEP)
def test_int8_engine_random_sweep(case):
    """Seeded sweep of the int8 digit engine (fp32 mode, 256 < h <= 1500): ragged tall / wide shapes,
    batches, input dtypes, scalings and ill-conditioned controlled spectra (singular values
    log-uniform down to 1e-5 or Pareto-like) against the oracle at the fp32-mode bar."""
    rng = np.random.default_rng(4000 + case)
    h = int(rng.integers(257, 1500))
    w = int(rng.integers(h, min(4096, 3 * h)))
    tall = rng.random() < 0.6
    batch = int(rng.choice([1, 1, 2]))
    dtype = {0: torch.float32, 1: torch.float32, 2: torch.float64, 3: torch.bfloat16}[int(rng.integers(0, 4))]
    scaling = str(rng.choice(["gram", "gram", "plain"]))
    ms = []
    for i in range(batch):
        if rng.random() < 0.5:
            s = np.exp(rng.uniform(np.log(1e-5), 0.0, h))
        else:
            s = 1.0 + rng.pareto(1.5, h)
            s = 1e-6 + (s - s.min()) / (s.max() - s.min())
        m = O.controlled_spectrum_matrix(w, h, s, 100 * case + i) if tall else \
            O.controlled_spectrum_matrix(h, w, s, 100 * case + i)
        ms.append(m)
    x = torch.from_numpy(np.stack(ms)).to(dtype).to(DEV)
    xin = x[0] if batch == 1 else x
    res = U.orthogonalize(xin, spec(scaling=scaling), precision="fp32")
    torch.cuda.synchronize()
    y = res.y.reshape(x.shape).double().cpu().numpy()
    src = x.double().cpu().numpy()
    worst = 0.0
    for i in range(batch):
        ref = O.run(src[i], "unso", scaling=scaling)["y"]
        worst = max(worst, rel(y[i], ref))
    tol = 1e-5 + (2.0 ** -9 if dtype == torch.bfloat16 else 0.0)
    print(f"case {case}: {x.shape} {str(dtype)[6:]} {scaling}: {worst:.2e}")
    assert worst <= tol


NS_CASES = [
    # (shape, method, iterations, dtype): the NS comparison path (ortho.py:209-233) in fp32 mode, h > 256
    ((1000, 333), "muon", 5, torch.float32),      # tall, ragged h
    ((300, 700), "muon", 5, torch.float64),       # wide, fp64 I/O
    ((2048, 512), "muon", 5, torch.float32),      # configs[1] matrix
    ((700, 300), "original", 6, torch.float32),   # cubic NS, tall
    ((520, 1100), "original", 8, torch.float32),  # cubic NS, wide
]


@pytest.mark.parametrize("case", range(len(NS_CASES)))
def test_int8_engine_ns_matches_oracle(case):
    """Newton-Schulz on the int8 digit engine: Gram of the state, the quintic operator b G + c G^2 and
    the state update per iteration, against the oracle's NS loop and against the fp64 DMMA engine."""
    shape, method, iters, dtype = NS_CASES[case]
    kind = U.MethodKind.MUON_NS if method == "muon" else U.MethodKind.ORIGINAL_NS
    m = controlled(*shape, 0.05, 70 + case)
    x = torch.from_numpy(m).to(dtype).to(DEV)
    res = U.orthogonalize(x, U.MethodSpec(kind, iterations=iters), precision="fp32")
    dm = U.orthogonalize(x, U.MethodSpec(kind, iterations=iters, fp32_engine="dmma"), precision="fp32")
    torch.cuda.synchronize()
    ref = O.run(x.double().cpu().numpy(), method, iterations=iters)["y"]
    y = res.y.double().cpu().numpy()
    e_or, e_dm = rel(y, ref), rel(y, dm.y.double().cpu().numpy())
    print(f"{shape} {method}-{iters}: vs oracle {e_or:.2e}, vs fp64 DMMA {e_dm:.2e}")
    assert e_or <= 1e-5
    assert e_dm <= 2e-6
