"""Dev tool: stress the persistent bf16 chain's one- and two-slot forms: random (h, w, batch) on that route,
repeated calls interleaved with other shapes; every batch result must be finite, bit-identical between
repeated calls, and agree with the fp32 mode (fp64-grade) on a sampled matrix.  usage: python tools/chain_stress.py [iters] [seed]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_02500_b200 as U  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = torch.Generator(device="cuda").manual_seed(seed)
rng = torch.Generator().manual_seed(seed)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
t0 = time.time()
worst = 0.0
for it in range(iters):
    h = int(torch.randint(129, 1100, (1,), generator=rng))
    if it % 7 == 0:
        h = int(torch.randint(1100, 2049, (1,), generator=rng))
    nt = (h + 127) // 128
    tpm = nt * (nt + 1) // 2
    bmax = max(1, min(40, (4 * 2 * (148 // tpm))))
    b = int(torch.randint(1, bmax + 1, (1,), generator=rng))
    w = h + int(torch.randint(0, 1500, (1,), generator=rng))
    x = torch.randn(b, w, h, generator=g, device="cuda")
    if it % 3 == 0:  # spread the spectra of some matrices so groups take different truncation decisions
        scale = torch.logspace(0, -3, h, device="cuda")
        x[b // 2:] = x[b // 2:] * scale
    xb = x.to(torch.bfloat16)
    y1 = U.orthogonalize(xb, spec, precision="bf16", check=False).y
    y2 = U.orthogonalize(xb, spec, precision="bf16", check=False).y
    torch.cuda.synchronize()
    assert torch.isfinite(y1).all(), (it, h, w, b)
    assert torch.equal(y1, y2), (it, h, w, b, "not deterministic")
    if it % 10 == 0:
        i = int(torch.randint(0, b, (1,), generator=rng))
        ref = U.orthogonalize(xb[i].float(), spec, precision="fp32").y
        r = float((y1[i].float() - ref).norm() / ref.norm())
        worst = max(worst, r)
        assert r <= 2e-2, (it, h, w, b, i, r)
print(f"chain_stress: {iters} iterations ok, worst sampled rel err vs fp32 mode {worst:.2e}, {time.time() - t0:.0f} s")
