"""Measure every BASELINE.json config on one B200 (supplement to bench.py's headline cfg4).

For each config: device time (CUDA events, warm), model TFLOP/s (kernel_model_flops),
matrices/s, % of the measured bf16 peak, and a consistency check of the bf16 result
against the fp32-mode (fp64-grade) device path on the same rounded input.  Inputs are
seeded synthetic data with BASELINE's shapes and distributions.

usage: python tools/bench_configs.py [--only cfg3,cfg5] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402

DEV = torch.device("cuda:0")
PEAK = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["bf16_tflops"] if os.path.exists(
    os.path.join(REPO, "MEASURED_PEAKS.json")) else 1590.0


def haar_cols(n, k, g):
    q, r = torch.linalg.qr(torch.randn(n, k, generator=g, device=DEV, dtype=torch.float64))
    return q * torch.sign(torch.diagonal(r))


def controlled(rows, cols, s, g):
    k = min(rows, cols)
    u = haar_cols(rows, k, g)
    v = haar_cols(cols, k, g)
    return (u * s[None, :]) @ v.T


def timed(fn, warm=1, reps=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm())


def ortho_pair(x0, y0, spec):
    """(ours, reference) orthogonality error ||Y^T Y - I||_F of matrix 0: ours from Y; the
    reference's from the scalar map of sigma(X) (Y_ref = X P(X^T X) has singular values g(sigma)),
    i.e. its exact-arithmetic value on the same input.  Spectra from fp64 Grams on the device."""
    def gram(z):
        z = z.double()
        return z.T @ z if z.shape[0] >= z.shape[1] else z @ z.T
    gy = gram(y0)
    ours = float((gy - torch.eye(gy.shape[0], device=gy.device, dtype=gy.dtype)).norm())
    sx = torch.sqrt(torch.linalg.eigvalsh(gram(x0)).clamp_min(0.0)).cpu().numpy()
    scale = float((sx ** 4).sum()) ** 0.25 if spec.effective_scaling is U.Scaling.FROBENIUS_GRAM else \
        float(np.sqrt((sx ** 2).sum()))
    sy = U.scalar_map(spec)(sx / scale)
    return ours, float(np.sqrt(((sy ** 2 - 1.0) ** 2).sum()))


def run(name, x, spec, precision, nmat, h, w, reps=3, check_against=None):
    ms = timed(lambda: U.orthogonalize(x, spec, precision=precision, check=False), reps=reps)
    f = U.kernel_model_flops(h, w, spec) * nmat
    out = {"config": name, "precision": precision, "ms": ms, "matrices_per_s": nmat / (ms / 1e3),
           "model_tflops": f / (ms / 1e3) / 1e12, "pct_bf16_peak": f / (ms / 1e3) / 1e12 / PEAK}
    res = U.orthogonalize(x, spec, precision=precision, check=True)
    if res.info:
        out["apply_single"] = [bool(i["apply_single"]) for i in res.info][:4]
    if check_against is not None:
        out["rel_vs_fp64_path"] = rel(res.y, check_against)
    x0 = x if x.dim() == 2 else x[0]
    y0 = res.y if res.y.dim() == 2 else res.y[0]
    out["ortho_error"], out["ortho_error_reference"] = ortho_pair(
        x0.to(torch.bfloat16) if precision == "bf16" else x0, y0, spec)
    print(json.dumps(out), flush=True)
    return out


def run_graphed(name, x, spec, precision, nmat, h, w, reps=50):
    from paper_2602_02500_b200.graphs import GraphedOrthogonalize
    g = GraphedOrthogonalize(x, spec, precision=precision)
    ms = timed(lambda: g(), warm=3, reps=reps)
    f = U.kernel_model_flops(h, w, spec) * nmat
    out = {"config": name + " (CUDA graph replay)", "precision": precision, "ms": ms,
           "matrices_per_s": nmat / (ms / 1e3), "model_tflops": f / (ms / 1e3) / 1e12}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    only = set(args.only.split(","))
    unso = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
    muon = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5)
    results = []
    g = torch.Generator(device=DEV).manual_seed(0)
    if "cfg1" in only:
        from oracle import unso_oracle as O  # checker only
        x = torch.from_numpy(O.gaussian_matrix(512, 128, 0).astype(np.float32)).to(DEV)
        ref = U.orthogonalize(x.double(), unso, precision="fp32").y
        refb = U.orthogonalize(x.to(torch.bfloat16).double(), unso, precision="fp32").y
        results.append(run("cfg1 512x128 unso", x, unso, "fp32", 1, 128, 512, reps=20, check_against=ref))
        results.append(run("cfg1 512x128 unso", x, unso, "bf16", 1, 128, 512, reps=20, check_against=refb))
        results.append(run("cfg1 512x128 muon5", x, muon, "fp32", 1, 128, 512, reps=20))
        for prec in ("fp32", "bf16"):
            results.append(run_graphed("cfg1 512x128 unso", x, unso, prec, 1, 128, 512))
        results.append(run_graphed("cfg1 512x128 muon5", x, muon, "fp32", 1, 128, 512))
    if "cfg2" in only:
        s = torch.exp(torch.empty(16, 512, device=DEV, dtype=torch.float64).uniform_(np.log(1e-4), 0.0, generator=g))
        x = torch.stack([controlled(2048, 512, s[i], g) for i in range(16)]).float()
        ref = U.orthogonalize(x.double(), unso, precision="fp32").y
        refb = U.orthogonalize(x.to(torch.bfloat16).double(), unso, precision="fp32").y  # same rounded input
        results.append(run("cfg2 16x2048x512 unso", x, unso, "fp32", 16, 512, 2048, check_against=ref))
        results.append(run("cfg2 16x2048x512 unso", x, unso, "bf16", 16, 512, 2048, check_against=refb))
        for prec in ("fp32", "bf16"):
            results.append(run_graphed("cfg2 16x2048x512 unso", x, unso, prec, 16, 512, 2048, reps=20))
    if "cfg3" in only:
        # one layer group: 4 layers x {4 x 4096^2} and 4 layers x {3 x 14336x4096}, N(0, 0.02^2), bf16
        xs = (torch.randn(16, 4096, 4096, generator=g, device=DEV) * 0.02).to(torch.bfloat16)
        xt = (torch.randn(12, 14336, 4096, generator=g, device=DEV) * 0.02).to(torch.bfloat16)
        ref = U.orthogonalize(xs[:1].double(), unso, precision="fp32").y
        a = run("cfg3 square 16x4096^2 unso", xs, unso, "bf16", 16, 4096, 4096, reps=2)
        a["rel_vs_fp64_path"] = rel(U.orthogonalize(xs[:1], unso, precision="bf16").y, ref)
        b = run("cfg3 tall 12x14336x4096 unso", xt, unso, "bf16", 12, 4096, 14336, reps=2)
        results += [a, b]
        tot_f = 128 * U.kernel_model_flops(4096, 4096, unso) + 96 * U.kernel_model_flops(4096, 14336, unso)
        tot_ms = a["ms"] / 16 * 128 + b["ms"] / 12 * 96
        print(json.dumps({"config": "cfg3 full 32 layers (extrapolated from the two groups)",
                          "ms": tot_ms, "model_tflops": tot_f / (tot_ms / 1e3) / 1e12,
                          "pct_bf16_peak": tot_f / (tot_ms / 1e3) / 1e12 / PEAK}), flush=True)
        del xs, xt
    if "cfg4" in only:
        x = torch.randn(262144, 2048, generator=g, device=DEV).to(torch.bfloat16)
        results.append(run("cfg4 262144x2048 unso", x, unso, "bf16", 1, 2048, 262144, reps=10))
        # the comparison path on the same input: 5 Muon-coefficient NS steps (reference-model FLOPs)
        results.append(run("cfg4 262144x2048 muon5", x, muon, "bf16", 1, 2048, 262144, reps=3))
        muon_fast = U.MethodSpec(U.MethodKind.MUON_NS, iterations=5, ns_products="bf16")
        results.append(run("cfg4 262144x2048 muon5 (single-bf16 state products)", x, muon_fast, "bf16", 1, 2048,
                           262144, reps=3))
        del x
    if "cfg5" in only:
        u = torch.rand(4, 8192, generator=g, device=DEV, dtype=torch.float64)
        s = 1.0 / (1.0 - u) ** (1.0 / 1.5)                     # classical Pareto(alpha=1.5), min 1
        s = 1e-6 + (s - s.min(1, keepdim=True).values) / (s.max(1, keepdim=True).values - s.min(1, keepdim=True).values) * (1 - 1e-6)
        x = torch.stack([controlled(16384, 8192, s[i], g) for i in range(4)]).float()
        ref = U.orthogonalize(x[:1].double(), unso, precision="fp32").y
        refb = U.orthogonalize(x[:1].to(torch.bfloat16).double(), unso, precision="fp32").y
        a = run("cfg5 4x16384x8192 unso", x, unso, "bf16", 4, 8192, 16384, reps=2)
        a["rel_vs_fp64_path"] = rel(U.orthogonalize(x[:1], unso, precision="bf16").y, refb)
        b = run("cfg5 1x16384x8192 unso", x[:1], unso, "fp32", 1, 8192, 16384, reps=1, check_against=ref)
        results += [a, b]
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(results, fh, indent=1)


if __name__ == "__main__":
    main()
