"""Dev tool: cfg1 (512x128 fp32, seed 0) orthogonalizations for launch lists: bf16 then fp32 mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_02500_b200 as U
from oracle import unso_oracle as O
x = torch.from_numpy(O.gaussian_matrix(512, 128, 0).astype(np.float32)).cuda()
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for prec in ("bf16", "fp32"):
    U.orthogonalize(x, spec, precision=prec, check=False)
torch.cuda.synchronize()
print("ok")
