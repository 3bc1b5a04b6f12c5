"""Stale-state regression tests: every call runs on a workspace pre-filled with 0xFF bytes (bf16
0xFFFF, e4m3 0xFF and f32/f64 0xFF.. are all NaN), so any kernel that reads a byte it did not
write in the same call -- padding columns of a ragged h, unused partial slots, a tile another
route owns -- turns the output into NaN (or garbage) instead of silently passing on a fresh,
zeroed allocation.  Covers every route of the boundary: the small on-chip chain (h <= 128), the
persistent chain (h <= 2048, batch chunks), the glue-free multi-launch route (h > 2048, e4m3 cross
terms and bf16x3), the legacy route (Gelfand scaling at large h), fp32 mode (fp64 DMMA engine) and
the NS comparison path in both modes.  Each output must be finite and within the mode's bar of the
CPU oracle (fp32 1e-5, bf16 2e-2 on the bf16-rounded input; + 2^-9 for a bf16 output).

The round-1 bug these pin: a ragged h > 2048 after a larger h in the same process
returned NaN, because the squaring epilogue re-emitted stale padding columns [h, ldc) into the
interleaved e4m3 operand, whose TMA map spans the padding (ortho.py:171-205 is the path)."""

import numpy as np
import pytest
import torch

import paper_2602_02500_b200 as U
from oracle import unso_oracle as O

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
TOL = {"fp32": 1e-5, "bf16": 2e-2}
POISON_BYTES = 768 << 20


def poison():
    """Give the pool a >= 768 MiB buffer for the current stream and fill it with 0xFF."""
    stream = torch.cuda.current_stream(DEV)
    buf = U.ortho.workspace_pool.get(POISON_BYTES, DEV, stream)
    buf.fill_(0xFF)
    torch.cuda.synchronize()


def spec_of(kind, **kw):
    if kind == "unso":
        return U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), **kw)
    if kind == "muon":
        return U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, **kw)
    if kind == "original":
        return U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=8, **kw)
    return U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=U.CesistaStepParams(U.default_cesista_triples()), **kw)


def oracle(m64, kind, scaling=None):
    if kind == "cesista":
        return O.run(m64, "cesista", rows=O.cesista_rows(O.CESISTA_DEFAULT_TRIPLES))["y"]
    if kind == "unso":
        return O.run(m64, "unso", scaling=scaling)["y"]
    return O.run(m64, kind)["y"]


def run_checked(shape, kind, precision, dtype, seed, std=0.02, **kw):
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = (torch.randn(*shape, generator=g, device=DEV) * std).to(dtype)
    poison()
    spec = spec_of(kind, **kw)
    res = U.orthogonalize(x, spec, precision=precision)
    torch.cuda.synchronize()
    y = res.y
    assert torch.isfinite(y).all(), (shape, kind, precision, "non-finite output on a poisoned workspace")
    src = (x.to(torch.bfloat16) if precision == "bf16" else x).double().cpu().numpy()
    got = y.double().cpu().numpy()
    if src.ndim == 2:
        src, got = src[None], got[None]
    tol = TOL[precision] + (2.0 ** -9 if dtype == torch.bfloat16 else 0.0)
    worst = 0.0
    for b in range(src.shape[0]):
        ref = oracle(src[b], kind, kw.get("scaling"))
        err = float(np.linalg.norm(got[b] - ref) / np.linalg.norm(ref))
        worst = max(worst, err)
    print(f"poisoned {shape} {kind} {precision} {str(dtype)[6:]} {kw}: {worst:.2e}")
    assert worst <= tol, (shape, kind, precision, kw, worst)
    return worst


ROUTES = [
    # (shape, kind, precision, dtype, extra spec keywords)
    ((512, 128), "unso", "bf16", torch.bfloat16, {}),             # small route, fused Gram
    ((300, 100), "unso", "bf16", torch.float32, {}),              # small route, ragged
    ((96, 700), "unso", "bf16", torch.bfloat16, {}),              # small route, wide
    ((3000, 1000), "unso", "bf16", torch.bfloat16, {}),           # persistent chain, ragged h
    ((1300, 2000), "unso", "bf16", torch.bfloat16, {}),           # persistent chain, wide ragged
    ((24, 900, 640), "unso", "bf16", torch.bfloat16, {}),         # persistent chain, batch chunks
    ((2475, 2128), "unso", "bf16", torch.bfloat16, {}),           # glue-free, e4m3 cross terms, ragged
    ((2100, 2200), "unso", "bf16", torch.bfloat16, {}),           # glue-free, wide, ragged
    ((2, 2339, 2422), "unso", "bf16", torch.bfloat16, {}),        # glue-free, batch, ragged
    ((2475, 2128), "unso", "bf16", torch.bfloat16, {"chain": "bf16x3"}),
    ((2400, 2200), "unso", "bf16", torch.bfloat16, {"scaling": "gelfand"}),  # legacy route
    ((2400, 2200), "unso", "bf16", torch.bfloat16, {"scaling": "plain"}),
    ((900, 333), "unso", "fp32", torch.float32, {}),              # fp64 DMMA engine, small chain
    ((2300, 2100), "unso", "fp32", torch.float32, {}),            # fp64 DMMA engine, large h
    ((700, 260), "unso", "fp32", torch.float32, {"scaling": "gelfand"}),
    ((1000, 300), "muon", "bf16", torch.bfloat16, {}),
    ((300, 1000), "muon", "bf16", torch.bfloat16, {"ns_products": "bf16"}),
    ((2200, 2100), "muon", "bf16", torch.bfloat16, {}),
    ((1000, 300), "original", "fp32", torch.float32, {}),
    ((640, 900), "cesista", "bf16", torch.bfloat16, {}),
    ((777, 555), "muon", "fp32", torch.float32, {}),
]


@pytest.mark.parametrize("case", range(len(ROUTES)))
def test_route_on_poisoned_workspace(case):
    shape, kind, precision, dtype, kw = ROUTES[case]
    run_checked(shape, kind, precision, dtype, 500 + case, **kw)


# The recorded round-1 failing sequences (tools/repro_large_h_nan.py): a smaller ragged h after a
# larger one, on a workspace left over by the larger call (no poisoning between the calls).
SEQUENCES = [
    [(2422, 2339), (2128, 2475)],
    [(2339, 2422), (2128, 2475)],
    [(2422, 2339), (2100, 2200)],
    [(4096, 2600), (2475, 2128), (2200, 2100)],
]


@pytest.mark.parametrize("seq", range(len(SEQUENCES)))
def test_decreasing_h_sequences(seq):
    U.ortho.workspace_pool.clear()
    torch.cuda.empty_cache()
    spec = spec_of("unso")
    for i, (r, c) in enumerate(SEQUENCES[seq]):
        g = torch.Generator(device=DEV).manual_seed(50 + i)
        x = (torch.randn(r, c, generator=g, device=DEV) * 0.02).to(torch.bfloat16)
        y = U.orthogonalize(x, spec).y
        torch.cuda.synchronize()
        assert torch.isfinite(y).all(), (seq, i, r, c)
        ref = O.run(x.double().cpu().numpy(), "unso")["y"]
        err = float(np.linalg.norm(y.double().cpu().numpy() - ref) / np.linalg.norm(ref))
        print(f"sequence {seq} call {i} {r}x{c}: {err:.2e}")
        assert err <= TOL["bf16"] + 2.0 ** -9, (seq, i, r, c, err)
