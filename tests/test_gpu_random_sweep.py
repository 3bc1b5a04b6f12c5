"""Seeded random sweep of the boundary against the oracle: random shapes (ragged, tall and wide,
1 <= h <= 1100, w <= 4096), batch sizes, methods, scalings, precisions and input dtypes, each case
checked at the mode's bar (relative Frobenius error <= 1e-5 in fp32 mode, <= 2e-2 in bf16 mode) on
the values the mode computes on (bf16 mode: the bf16-rounded input).  Complements the hand-picked
cases of test_gpu_parity / test_gpu_edge_cases with combinations nobody chose."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
BAR = {"fp32": 1e-5, "bf16": 2e-2}


def _spec(rng):
    kind = rng.choice(["unso", "unso", "unso", "muon", "original", "cesista"])
    if kind == "unso":
        scaling = str(rng.choice(["gram", "plain", "gelfand"]))
        return U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling=scaling), "unso", scaling
    if kind == "muon":
        return U.MethodSpec(U.MethodKind.MUON_NS, iterations=5), "muon", None
    if kind == "original":
        return U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=8), "original", None
    return (U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=U.CesistaStepParams(U.default_cesista_triples())),
            "cesista", None)


def _oracle(m64, spec, kind, scaling):
    if kind == "unso":
        return O.run(m64, "unso", scaling=scaling)["y"]
    if kind == "cesista":
        return O.run(m64, "cesista", rows=O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES))["y"]
    return O.run(m64, kind)["y"]


CASES = list(range(64))


@pytest.mark.parametrize("case", CASES)
def test_random_case(case):
    rng = np.random.default_rng(1000 + case)
    h = int(rng.choice([int(rng.integers(1, 130)), int(rng.integers(130, 600)), int(rng.integers(600, 1100))]))
    w = int(rng.integers(h, max(h + 1, min(4096, 4 * h + 64))))
    rows, cols = (w, h) if rng.random() < 0.5 else (h, w)
    batch = int(rng.choice([1, 1, 2, 3]))
    precision = str(rng.choice(["fp32", "bf16"]))
    dtype = torch.bfloat16 if (precision == "bf16" and rng.random() < 0.7) else torch.float32
    spec, kind, scaling = _spec(rng)
    g = torch.Generator(device=DEV).manual_seed(case)
    x = torch.randn(batch, rows, cols, generator=g, device=DEV) * float(rng.choice([1.0, 0.02, 30.0]))
    x = x.to(dtype)
    xin = x[0] if batch == 1 else x
    res = U.orthogonalize(xin, spec, precision=precision)
    y = res.y.reshape(batch, rows, cols)
    assert y.dtype == dtype and y.shape == (batch, rows, cols)
    src = x.to(torch.bfloat16) if precision == "bf16" else x
    for b in range(batch):
        m64 = src[b].double().cpu().numpy()
        ref = _oracle(m64, spec, kind, scaling)
        got = y[b].double().cpu().numpy()
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"case {case}: {rows}x{cols} b{batch} {precision} {str(dtype)[6:]} {kind}/{scaling}: {err:.2e}")
        assert err <= BAR[precision], (case, rows, cols, batch, precision, str(dtype), kind, scaling, err)



# Large-h sweep: ragged h in (2048, 4608] (the multi-launch glue-free route with e4m3 cross terms,
# h % 256 != 0), tall and wide, run as ONE decreasing-h call sequence in a single process with the
# pooled workspace left over from the previous (larger) call -- the order that exposed the round-1
# stale-padding NaN.  Each output is checked against the oracle.
def _large_h_cases():
    rng = np.random.default_rng(4242)
    cases = []
    for i in range(8):
        lo, hi = (4097, 4608) if i == 0 else (2049, 4608 if i < 3 else 3200)
        h = int(rng.integers(lo, hi + 1))
        if h % 256 == 0:
            h += 7
        w = int(rng.integers(h, h + 600))
        tall = bool(rng.random() < 0.5)
        kind = str(rng.choice(["unso", "unso", "unso", "muon"]))
        precision = "bf16" if (kind == "muon" or rng.random() < 0.8) else "fp32"
        cases.append((h, w, tall, kind, precision))
    return sorted(cases, key=lambda c: -c[0])


def test_large_h_decreasing_sequence():
    for i, (h, w, tall, kind, precision) in enumerate(_large_h_cases()):
        rows, cols = (w, h) if tall else (h, w)
        dtype = torch.bfloat16 if precision == "bf16" else torch.float32
        g = torch.Generator(device=DEV).manual_seed(9000 + i)
        x = (torch.randn(rows, cols, generator=g, device=DEV) * 0.02).to(dtype)
        spec = (U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients()) if kind == "unso"
                else U.MethodSpec(U.MethodKind.MUON_NS, iterations=5))
        y = U.orthogonalize(x, spec, precision=precision).y
        torch.cuda.synchronize()
        assert torch.isfinite(y).all(), (i, rows, cols, kind, precision)
        ref = O.run(x.double().cpu().numpy(), kind)["y"]
        err = float(np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref))
        print(f"large-h {i}: {rows}x{cols} {kind} {precision}: {err:.2e}")
        tol = BAR[precision] + (2.0 ** -9 if dtype == torch.bfloat16 else 0.0)
        assert err <= tol, (i, rows, cols, kind, precision, err)
