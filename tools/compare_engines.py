"""Dev tool: run one configuration in a fresh process and dump Y for cross-engine comparison."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2602_02500_b200 as U

rows, cols, prec, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
g = torch.Generator(device="cuda").manual_seed(1234)
x = torch.randn(rows, cols, generator=g, device="cuda").to(torch.bfloat16)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
xin = x if prec == "bf16" else x.double()
res = U.orthogonalize(xin, spec, precision=prec)
torch.cuda.synchronize()
y = res.y.float()
print(prec, os.environ.get("UNSO_ENGINE", "pair"), "ortho_error", U.ortho_error_any(res.y))
torch.save(y.cpu(), out)
