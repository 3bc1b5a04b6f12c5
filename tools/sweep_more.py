"""Dev tool: extra seeded sweeps against the oracle beyond the committed test cases.
  part 1: tests/test_gpu_random_sweep.test_random_case for case ids [lo, hi) (new random combinations)
  part 2: bf16 UNSO batches that run the persistent chain in its two-slot form (batch 8-40, 129 <= h <= 1100,
          mixed well- / ill-conditioned matrices), every matrix against the oracle.
usage: python tools/sweep_more.py [lo] [hi] [batch_cases]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2602_02500_b200 as U  # noqa: E402
from oracle import unso_oracle as O  # noqa: E402  (checker)
import test_gpu_random_sweep as S  # noqa: E402

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 64
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 300
nb_cases = int(sys.argv[3]) if len(sys.argv) > 3 else 40
t0 = time.time()
bad = []
for case in range(lo, hi):
    try:
        S.test_random_case(case)
    except Exception as e:  # noqa: BLE001
        bad.append((case, repr(e)[:200]))
print(f"part 1: cases {lo}..{hi - 1}: {hi - lo - len(bad)} ok, {len(bad)} failed, {time.time() - t0:.0f} s")
for b in bad:
    print("   FAILED", b)

spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
worst, bad2 = 0.0, []
t0 = time.time()
for case in range(nb_cases):
    rng = np.random.default_rng(5000 + case)
    h = int(rng.integers(129, 1101))
    w = h + int(rng.integers(0, 1200))
    nt = (h + 127) // 128
    tpm = nt * (nt + 1) // 2
    b_lo = min(max(2, 148 // tpm + 1), 39)  # more tiles than one wave of CTAs holds, where a batch of <= 40 can
    b = int(rng.integers(b_lo, max(b_lo + 1, min(40, 4 * (148 // tpm)) + 1)))
    g = torch.Generator(device="cuda").manual_seed(case)
    x = torch.randn(b, w, h, generator=g, device="cuda")
    for i in range(b):
        if rng.random() < 0.5:
            x[i] *= torch.logspace(0, -float(rng.integers(1, 5)), h, device="cuda")
    tall = rng.random() < 0.7
    xb = (x if tall else x.transpose(1, 2).contiguous()).to(torch.bfloat16)
    y = U.orthogonalize(xb, spec, precision="bf16").y
    torch.cuda.synchronize()
    for i in range(b):
        ref = O.run(xb[i].double().cpu().numpy(), "unso")["y"]
        r = float(np.linalg.norm(y[i].double().cpu().numpy() - ref) / np.linalg.norm(ref))
        worst = max(worst, r)
        if not (r <= 2e-2 + 2.0 ** -9):
            bad2.append((case, h, w, b, i, r))
print(f"part 2: {nb_cases} batches: worst rel err {worst:.2e}, {len(bad2)} matrices over the bar, {time.time() - t0:.0f} s")
for b in bad2[:20]:
    print("   FAILED", b)
sys.exit(1 if (bad or bad2) else 0)
