"""CPU emulation of the Muon-5 bf16 products (operand rounding emulated, fp64 accumulation): which of the
state-touching long-side products (Gram of X_k, update X_k B) needs the hi/lo state.  Dev tool; see DESIGN.md §2."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import unso_oracle as O
def bf16(a): return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).double().numpy()
def split(a):
    h = bf16(a); return h, bf16(a - h)
rows = O.muon_rows(5)
def muon(x, gram_mode, apply_mode):
    x = x / np.linalg.norm(x)
    x = x.T if x.shape[0] > x.shape[1] else x   # row-wide h x w
    for a, b, c in rows:
        xg = {"exact": x, "bf16": bf16(x), "x3": None}[gram_mode]
        if gram_mode == "x3":
            h, l = split(x); G = h @ h.T + h @ l.T + l @ h.T
        else:
            G = xg @ xg.T
        G = G.astype(np.float32).astype(np.float64)
        B = b * G + c * G @ G
        bh, bl = split(B)
        if apply_mode == "exact": XB = B @ x
        elif apply_mode == "bf16": XB = (bh + bl) @ bf16(x)
        else:
            h, l = split(x); XB = bh @ h + bl @ h + bh @ l
        x = (a * x + XB).astype(np.float32).astype(np.float64)
    return x
for name, m in [("gauss 1024x256", O.gaussian_matrix(1024, 256, 1)), ("gauss 512x512", O.gaussian_matrix(512, 512, 2))]:
    m = bf16(m)
    ref = muon(m, "exact", "exact")
    for g, ap in [("bf16", "bf16"), ("bf16", "exact"), ("exact", "bf16"), ("x3", "bf16"), ("bf16", "x3"), ("x3", "x3")]:
        y = muon(m, g, ap)
        print(f"{name} gram={g:5s} apply={ap:5s}: rel {np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}")
