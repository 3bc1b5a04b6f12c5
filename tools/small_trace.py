"""Dev tool: phase timeline of chain_small_kernel (build with -DUNSO_EXP_TIMING, load via UNSO_LIB)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402
from paper_2602_02500_b200 import _native as N  # noqa: E402

x = torch.randn(512, 128, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for _ in range(3):
    U.orthogonalize(x, spec, precision="bf16", check=False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 64 * 5))()
assert N.lib().unso_debug_chain_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(3, 64, 5).astype(np.float64)[0]
t0 = t[0, 0]
a = t[60]
print("phase A detail (us from start): partial sums %.2f, barrier %.2f, C tile stored %.2f, norms reduced %.2f"
      % tuple((a[i] - t0) / 1e3 for i in range(4)))
print(f"phase A: {(t[0, 1] - t0) / 1e3:.2f} us")
prev = t[0, 1]
for k in range(1, 14):
    if t[k, 3] == 0 or t[k, 3] < t0:
        continue
    print(f"step {k:2d}: mma {(t[k, 3] - prev) / 1e3:6.2f}  epilogue {(t[k, 4] - t[k, 3]) / 1e3 if t[k, 4] > t[k, 3] else float('nan'):6.2f} us")
    prev = t[k, 4] if t[k, 4] > t[k, 3] else t[k, 3]
print(f"final: {(t[0, 2] - prev) / 1e3:.2f} us; kernel total {(t[0, 2] - t0) / 1e3:.2f} us")
