"""Dev tool: per-step phase timeline of the persistent chain kernel (build with -DUNSO_EXP_TIMING,
load through UNSO_LIB).  usage: UNSO_LIB=exp/timing.so python tools/chain_trace.py [h] [rows] [batch]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402
from paper_2602_02500_b200 import _native as N  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
w = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
b = int(sys.argv[3]) if len(sys.argv) > 3 else 1
x = torch.randn(b, w, h, device="cuda").to(torch.bfloat16)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
for _ in range(3):
    U.orthogonalize(x, spec, check=False)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * 64 * 5))()
assert N.lib().unso_debug_chain_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(3, 64, 5).astype(np.float64)
for c in range(3):
    print(f"CTA slot {c}: step  first_data  mainloop  drain  epilogue  barrier   (us)")
    for k in range(1, 14):
        e = t[c, k]
        if e[0] == 0:
            continue
        nxt = t[c, k + 1, 0] if t[c, k + 1, 0] else np.nan
        print(f"   {k:2d}  {(e[1]-e[0])/1e3:8.2f}  {(e[2]-e[1])/1e3:8.2f}  {(e[3]-e[2])/1e3:6.2f}  "
              f"{(e[4]-e[3])/1e3:8.2f}  {(nxt-e[4])/1e3:7.2f}")
for c in range(3):
    a, f = t[c, 0], t[c, 63]
    if a[0] and f[0]:
        print(f"CTA slot {c}: phase A: partials+norms {(a[1]-a[0])/1e3:.2f} us, norm barrier {(a[2]-a[1])/1e3:.2f}, "
              f"C_1/P init {(a[3]-a[2])/1e3:.2f} (of which the norm sum {(a[4]-a[2])/1e3:.2f}); step 1 data after C_1 {(t[c,1,1]-a[3])/1e3:.2f}; "
              f"final: stats {(f[1]-f[0])/1e3:.2f}, barrier {(f[2]-f[1])/1e3:.2f}, P split+mirror {(f[3]-f[2])/1e3:.2f}; "
              f"kernel span {(f[3]-a[0])/1e3:.2f} us")

# per-k-block arrival timeline of CTA 0, squaring 5 (full-stage seen by the MMA issuer, stage freed for
# the producer), relative to the first arrival
kb = (ctypes.c_ulonglong * 128)()
if hasattr(N.lib(), "unso_debug_chain_kb") and N.lib().unso_debug_chain_kb(kb) == 0:
    a = np.frombuffer(kb, dtype=np.uint64).reshape(2, 64).astype(np.float64)
    full, free = a[0], a[1]
    n = int((full > 0).sum())
    t0 = full[0]
    print("squaring 5, CTA 0: k-block  full_at(us)  gap(us)  producer_free_at(us)")
    for kt in range(n):
        gap = (full[kt] - full[kt - 1]) / 1e3 if kt else 0.0
        print(f"   {kt:3d}  {(full[kt]-t0)/1e3:8.2f}  {gap:6.2f}  {(free[kt]-t0)/1e3 if free[kt] else float('nan'):8.2f}")
