"""Dev tool: per-tile timeline of one int8 digit-engine launch (pair 0), from a -DUNSO_EXP_TIMING build.
usage: UNSO_LIB=exp/timing.so python tools/oz_trace.py [batch rows cols] -- traces the LAST oz_gemm launch
of an fp32-mode orthogonalization (the apply)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402
from paper_2602_02500_b200 import _native as N  # noqa: E402

b, r, c = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16, 2048, 512)
x = torch.randn(b, r, c, device="cuda")
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for _ in range(2):
    U.orthogonalize(x, spec, precision="fp32")
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 16 * 8))()
assert N.lib().unso_debug_oz_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 16, 8).astype(np.float64)
for cta in range(2):
    t0 = t[cta, 15, 0]
    print(f"CTA {cta}: setup {(t[cta, 15, 1] - t0) / 1e3:.2f} us")
    for k in range(15):
        e = t[cta, k]
        if e[4] == 0:
            continue
        f = lambda v: (v - t0) / 1e3 if v else float('nan')
        print(f"  tile {k}: mma start {f(e[2]):8.2f}  mma issued {f(e[3]):8.2f}  epi tfull {f(e[4]):8.2f}  "
              f"released {f(e[5]):8.2f}  scales {f(e[0]) if k < 15 else 0:8.2f}  converted {f(e[1]) if k < 15 else 0:8.2f}  "
              f"done {f(e[6]):8.2f}")
