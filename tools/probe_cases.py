"""Dev tool: run small bf16 UNSO cases one per subprocess with a timeout; report hangs."""
import subprocess, sys, os
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys; sys.path.insert(0, {repo!r})
import numpy as np, torch
import paper_2602_02500_b200 as U
from oracle import unso_oracle as O
r, c, scaling, terms = {r}, {c}, {scaling!r}, {terms}
m = O.gaussian_matrix(r, c, r * 1000 + c).astype(np.float32)
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients(), scaling=scaling, apply_terms=terms)
res = U.orthogonalize(torch.from_numpy(m).cuda().to(torch.bfloat16), spec, precision="bf16")
torch.cuda.synchronize()
print("ok", res.info[0]["apply_single"] if res.info else None)
'''
for (r, c) in [(16, 40), (40, 16), (24, 24), (7, 13), (130, 66), (64, 256)]:
    for scaling in ("gram", "plain"):
        for terms in (None, 2, 1):
            code = CASE.format(repo=REPO, r=r, c=c, scaling=scaling, terms=terms)
            try:
                out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
                print(r, c, scaling, terms, out.stdout.strip()[-40:], out.stderr.strip()[-200:], flush=True)
            except subprocess.TimeoutExpired:
                print(r, c, scaling, terms, "HANG", flush=True)
