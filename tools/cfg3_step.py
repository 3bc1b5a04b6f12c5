"""Dev tool: one cfg3 square group (16 x 4096^2 bf16) orthogonalization, for launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_02500_b200 as U
g = torch.Generator(device="cuda").manual_seed(0)
x = (torch.randn(int(sys.argv[1]) if len(sys.argv) > 1 else 16, 4096, 4096, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
U.orthogonalize(x, spec, check=False)
torch.cuda.synchronize()
print("ok")
