"""Dev tool: per-step phase timeline of chain_f64_kernel (build with -DUNSO_EXP_TIMING, load via UNSO_LIB)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402
from paper_2602_02500_b200 import _native as N  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 128
x = torch.randn(4 * h, h, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for _ in range(3):
    U.orthogonalize(x, spec, precision="fp32", check=False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 64 * 5))()
assert N.lib().unso_debug_chain_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(3, 64, 5).astype(np.float64)
for c in range(3):
    print(f"CTA slot {c}: step  load  mma  epilogue  ->next step (us)")
    for k in range(1, 14):
        e = t[c, k]
        if e[0] == 0:
            continue
        nxt = t[c, k + 1, 0] if t[c, k + 1, 0] else np.nan
        print(f"   {k:2d}  {(e[1]-e[0])/1e3:5.2f} {(e[2]-e[1])/1e3:5.2f} {(e[3]-e[2])/1e3:6.2f}  {(nxt-e[3])/1e3:6.2f}")
