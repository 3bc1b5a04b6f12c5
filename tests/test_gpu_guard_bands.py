"""Out-of-bounds checks without compute-sanitizer (closed on this GPU pool): every route of the C ABI
runs with its output Y and its workspace placed between guard bands of a canary byte pattern, and its
input X inside a canary-filled buffer.  After the call the guard bytes must be untouched (no write
past Y or past the workspace size unso_workspace_size reported, in either direction) and X must be
unchanged (the library never writes its input).  The workspace itself is pre-filled with the canary,
so a route that reads bytes it did not write turns them into garbage the parity tests would catch
(tests/test_gpu_poisoned_workspace.py covers that side with NaN poisoning)."""

import ctypes

import pytest
import torch

import paper_2602_02500_b200 as U
from paper_2602_02500_b200 import _native as N
from paper_2602_02500_b200 import ortho as Ot

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0")
GUARD = 1 << 20  # bytes on each side
CANARY = 0xA5


def spec_of(kind, **kw):
    if kind == "unso":
        return U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), **kw)
    if kind == "muon":
        return U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, **kw)
    return U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=6, **kw)


ROUTES = [
    ((512, 128), "unso", "bf16", torch.bfloat16, {}),          # small on-chip chain, fused Gram
    ((300, 100), "unso", "bf16", torch.float32, {}),           # small chain, ragged, bf16 copy of X
    ((3000, 1000), "unso", "bf16", torch.bfloat16, {}),        # persistent chain, ragged
    ((5, 700, 640), "unso", "bf16", torch.bfloat16, {}),       # persistent chain, batch
    ((2475, 2128), "unso", "bf16", torch.bfloat16, {}),        # glue-free large-h chain (e4m3 cross terms)
    ((2128, 2475), "unso", "bf16", torch.bfloat16, {"chain": "bf16x3"}),
    ((2400, 2200), "unso", "bf16", torch.bfloat16, {"scaling": "gelfand"}),  # legacy route
    ((900, 200), "unso", "fp32", torch.float32, {}),           # fp64 cooperative chain (h <= 256)
    ((1000, 333), "unso", "fp32", torch.float32, {}),          # int8 digit engine, tall ragged
    ((300, 700), "unso", "fp32", torch.float64, {}),           # int8 digit engine, wide, fp64 I/O
    ((3, 600, 520), "unso", "fp32", torch.float32, {}),        # int8 digit engine, batch
    ((1000, 333), "unso", "fp32", torch.float32, {"fp32_engine": "dmma"}),
    ((1000, 300), "muon", "bf16", torch.bfloat16, {}),         # NS comparison path, bf16
    ((700, 300), "original", "fp32", torch.float32, {}),       # NS comparison path, fp32, int8 engine
    ((333, 1000), "muon", "fp32", torch.float64, {}),          # NS quintic, int8 engine, wide ragged
    ((2, 600, 520), "muon", "fp32", torch.float32, {}),        # NS quintic, int8 engine, batch
    ((700, 300), "muon", "fp32", torch.float32, {"fp32_engine": "dmma"}),
]


def guarded(nbytes):
    """A canary-filled uint8 buffer with `nbytes` usable bytes at a 256-aligned offset GUARD."""
    buf = torch.full((GUARD + nbytes + GUARD,), CANARY, dtype=torch.uint8, device=DEV)
    return buf, buf[GUARD:GUARD + nbytes]


def intact(buf, nbytes):
    return bool((buf[:GUARD] == CANARY).all()) and bool((buf[GUARD + nbytes:] == CANARY).all())


@pytest.mark.parametrize("case", range(len(ROUTES)))
def test_route_writes_stay_in_bounds(case):
    shape, kind, precision, dtype, kw = ROUTES[case]
    g = torch.Generator(device=DEV).manual_seed(900 + case)
    x = (torch.randn(*shape, generator=g, device=DEV) * 0.02).to(dtype)
    xd = Ot._matrix_desc(x)
    spec = spec_of(kind, **kw)
    md, co = Ot._method_desc(spec, U.Precision(precision), Ot._SCALING[spec.effective_scaling])
    lib = N.lib()
    ws_bytes = lib.unso_workspace_size(ctypes.byref(xd), ctypes.byref(md))
    assert ws_bytes > 0
    ws_bytes = (ws_bytes + 255) // 256 * 256
    xb = x.numel() * x.element_size()
    xbuf, xs = guarded(xb)
    xs.copy_(x.reshape(-1).view(torch.uint8))
    xin = xs.view(dtype).view(x.shape)
    ybuf, ys = guarded(xb)
    wbuf, ws = guarded(ws_bytes)
    before = xin.clone()
    stream = torch.cuda.current_stream(DEV)
    status = torch.zeros(xd.batch, dtype=torch.int32, device=DEV)
    code = lib.unso_orthogonalize(ctypes.byref(xd), ctypes.c_void_p(xin.data_ptr()), ctypes.c_void_p(ys.data_ptr()),
                                  ctypes.byref(md), ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws_bytes),
                                  ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    del co
    assert code == N.OK, code
    assert int(status.abs().sum()) == 0
    assert intact(ybuf, xb), f"{shape} {kind} {precision} {kw}: write outside Y"
    assert intact(wbuf, ws_bytes), f"{shape} {kind} {precision} {kw}: write outside the workspace"
    assert intact(xbuf, xb), f"{shape} {kind} {precision} {kw}: write around X"
    assert torch.equal(xin.reshape(-1).view(torch.uint8), before.reshape(-1).view(torch.uint8)), \
        "input X was modified"
    y = ys.view(dtype).view(x.shape)
    assert torch.isfinite(y).all()
