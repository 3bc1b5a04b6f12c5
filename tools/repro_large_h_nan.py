"""Reproduction of the open large-h bug (DESIGN.md §11 item 0): python tools/repro_large_h_nan.py 2422x2339 2128x2475
(bf16 UNSO on the multi-launch route: the second, smaller ragged h returns NaN)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_02500_b200 as U
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
shapes = [(int(a), int(b)) for a, b in (s.split("x") for s in sys.argv[1:])]
for i, (r, c) in enumerate(shapes):
    g = torch.Generator(device="cuda").manual_seed(50 + i)
    x = (torch.randn(r, c, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    y = U.orthogonalize(x, spec).y
    print(os.environ.get("UNSO_CHAIN_CROSS_ALL"), r, c, "NAN" if torch.isnan(y).any() else "ok", flush=True)
