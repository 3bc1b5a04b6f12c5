"""Run every route of the boundary once at small shapes, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_routes.py [filter]

Covers: the small on-chip chain (h <= 128), the persistent chain (ragged h, batch chunks), the
glue-free multi-launch large-h route (e4m3 cross terms and bf16x3), the legacy route (Gelfand /
plain scaling), the fp32 mode's fp64 DMMA engine (cooperative small chain and the tiled chain),
the NS comparison path in both modes, the row-sharded stages (unso_gram + unso_orthogonalize_from_gram),
the emulated NVLink peer Gram reduction (unso_gram_push / _reduce / _wait), the Muon multi-tensor
passes and the ortho-error kernel.  Outputs are only checked for finiteness here: parity is the test
suite's job; this script exists so the sanitizers see every kernel with a workspace it did not zero.
"""

from __future__ import annotations

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02500_b200 as U  # noqa: E402
from paper_2602_02500_b200 import distributed as D  # noqa: E402

DEV = torch.device("cuda:0")


def spec_of(kind, **kw):
    if kind == "unso":
        return U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), **kw)
    if kind == "muon":
        return U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, **kw)
    if kind == "original":
        return U.MethodSpec(U.MethodKind.ORIGINAL_NS, iterations=8, **kw)
    return U.MethodSpec(U.MethodKind.CESISTA_NS, step_params=U.CesistaStepParams(U.default_cesista_triples()), **kw)


ROUTES = [
    ("small", (512, 128), "unso", "bf16", torch.bfloat16, {}),
    ("small-ragged", (300, 100), "unso", "bf16", torch.float32, {}),
    ("small-wide", (96, 700), "unso", "bf16", torch.bfloat16, {}),
    ("persistent", (3000, 1000), "unso", "bf16", torch.bfloat16, {}),
    ("persistent-batch", (6, 900, 640), "unso", "bf16", torch.bfloat16, {}),
    ("persistent-2048", (4096, 2048), "unso", "bf16", torch.bfloat16, {}),
    ("gluefree-e4m3", (2475, 2128), "unso", "bf16", torch.bfloat16, {}),
    ("gluefree-bf16x3", (2475, 2128), "unso", "bf16", torch.bfloat16, {"chain": "bf16x3"}),
    ("legacy-gelfand", (2400, 2200), "unso", "bf16", torch.bfloat16, {"scaling": "gelfand"}),
    ("fp32-small", (900, 200), "unso", "fp32", torch.float32, {}),
    ("fp32-tiled", (1200, 700), "unso", "fp32", torch.float32, {}),
    ("ns-bf16", (1000, 300), "muon", "bf16", torch.bfloat16, {}),
    ("ns-bf16-single", (300, 1000), "muon", "bf16", torch.bfloat16, {"ns_products": "bf16"}),
    ("ns-fp32", (777, 555), "muon", "fp32", torch.float32, {}),
    ("original-fp32", (1000, 300), "original", "fp32", torch.float32, {}),
    ("cesista-bf16", (640, 900), "cesista", "bf16", torch.bfloat16, {}),
]


def poison():
    stream = torch.cuda.current_stream(DEV)
    U.ortho.workspace_pool.get(256 << 20, DEV, stream).fill_(0xFF)


def run_routes(flt):
    for name, shape, kind, precision, dtype, kw in ROUTES:
        if flt and flt not in name:
            continue
        g = torch.Generator(device=DEV).manual_seed(len(name))
        x = (torch.randn(*shape, generator=g, device=DEV) * 0.02).to(dtype)
        poison()
        t = time.time()
        y = U.orthogonalize(x, spec_of(kind, **kw), precision=precision).y
        torch.cuda.synchronize()
        ok = bool(torch.isfinite(y).all())
        print(f"[route] {name} {shape} {kind} {precision}: finite={ok} ({time.time() - t:.1f} s)", flush=True)
        assert ok, name


def run_sharded(flt):
    if flt and flt not in "sharded nvlink":
        return
    h, world = 512, 3
    g = torch.Generator(device=DEV).manual_seed(5)
    x = torch.randn(8 * h, h, generator=g, device=DEV).to(torch.bfloat16)
    spec = spec_of("unso")
    shards = [x[slice(*D.row_shard_bounds(x.shape[0], world, r))] for r in range(world)]
    gsum = sum(D.native_gram(s, spec, "bf16") for s in shards)
    ys = [D.native_finish(s, gsum.clone(), spec, "bf16")[0] for s in shards]
    torch.cuda.synchronize()
    print(f"[route] sharded stages world={world}: finite={all(bool(torch.isfinite(y).all()) for y in ys)}", flush=True)
    splits = D.gram_push_splits(h, min(s.shape[0] for s in shards))
    reducers = D.NvlinkGramReducer.emulated(h, world, splits, DEV)
    for r in range(world):
        reducers[r].push(shards[r], spec, "bf16")
    for r in range(world):
        reducers[r].reduce()
    gs = [reducers[r].wait() for r in range(world)]
    torch.cuda.synchronize()
    print(f"[route] nvlink emulated world={world}: equal={all(torch.equal(gs[0], q) for q in gs)}", flush=True)


def run_muon(flt):
    if flt and flt not in "muon-optimizer":
        return
    params = [torch.nn.Parameter(torch.zeros(256, 192, device=DEV, dtype=torch.bfloat16)) for _ in range(3)]
    opt = U.Muon(params, lr=0.02)
    for p in params:
        p.grad = torch.randn_like(p) * 0.02
    opt.step()
    torch.cuda.synchronize()
    print(f"[route] muon-optimizer: finite={all(bool(torch.isfinite(p).all()) for p in params)}", flush=True)


def run_error(flt):
    if flt and flt not in "ortho-error":
        return
    x = torch.randn(700, 300, device=DEV)
    e = U.ortho_error(x)
    print(f"[route] ortho-error: {float(e):.4f}", flush=True)


if __name__ == "__main__":
    flt = sys.argv[1] if len(sys.argv) > 1 else ""
    run_routes(flt)
    run_sharded(flt)
    run_muon(flt)
    run_error(flt)
    print("[sanitize_routes] done", flush=True)
