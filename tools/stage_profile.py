"""Dev tool: per-stage device times (library CUDA events) of one orthogonalize call per config.

usage: python tools/stage_profile.py cfg5b|cfg5f|cfg3s|cfg3t|cfg2b|cfg2f|cfg1b|cfg1f|cfg4 [reps] [batch]
Prints stage ms and model TFLOP/s of each stage's share (gram: 2wh^2, chain: 2(N-1)h^3, apply 2wh^2).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402
from paper_2602_02500_b200._native import PROFILE_STAGES, StageProfiler  # noqa: E402

CASES = {
    "cfg1b": (1, 512, 128, torch.float32, "bf16"), "cfg1f": (1, 512, 128, torch.float32, "fp32"),
    "cfg2b": (16, 2048, 512, torch.float32, "bf16"), "cfg2f": (16, 2048, 512, torch.float32, "fp32"),
    "cfg3s": (16, 4096, 4096, torch.bfloat16, "bf16"), "cfg3t": (12, 14336, 4096, torch.bfloat16, "bf16"),
    "cfg4": (1, 262144, 2048, torch.bfloat16, "bf16"),
    "cfg5b": (4, 16384, 8192, torch.float32, "bf16"), "cfg5f": (1, 16384, 8192, torch.float32, "fp32"),
}


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    b, w, h, dt, prec = CASES[name]
    if len(sys.argv) > 3:
        b = int(sys.argv[3])
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(b, w, h, generator=g, device="cuda").to(dt)
    chain = os.environ.get("UNSO_CHAIN")  # e.g. "bf16x3"
    truncate = os.environ.get("UNSO_TRUNCATE", "1") != "0"
    spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), chain=chain, truncate=truncate)
    U.orthogonalize(x, spec, precision=prec, check=False)
    torch.cuda.synchronize()
    with StageProfiler(reps) as prof:
        for _ in range(reps):
            U.orthogonalize(x, spec, precision=prec, check=False)
        torch.cuda.synchronize()
        t = prof.read()
    med = t[len(t) // 2] if len(t) else t
    fl = {"gram": 2.0 * w * h * h * b, "chain": 2.0 * 12 * h ** 3 * b, "apply": 2.0 * w * h * h * b}
    out = {"case": name, "precision": prec, "total_ms": float(med.sum())}
    info = U.orthogonalize(x, spec, precision=prec, check=True).info
    if info:
        out["chain_steps"] = info[0].get("chain_steps")
    for s, v in zip(PROFILE_STAGES, med):
        out[s + "_ms"] = round(float(v), 4)
        if s in fl and v > 0:
            out[s + "_tflops"] = round(fl[s] / (float(v) * 1e-3) / 1e12, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
