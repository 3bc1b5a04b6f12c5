"""Dev tool: error vs the oracle of the bf16-mode persistent chain on configs[1]- and configs[4]-like
spectra (2048 x 512) and a Gaussian 4096 x 1024, for the current UNSO_PCHAIN_HI_ONLY setting
(developer build).  usage: UNSO_LIB=exp/dev.so UNSO_PCHAIN_HI_ONLY=3 python tools/hi_only_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_02500_b200 as U  # noqa: E402
from oracle import unso_oracle as O  # noqa: E402

rng = np.random.default_rng(0)
cases = {
    "cfg2-like logU[1e-4,1]": O.controlled_spectrum_matrix(2048, 512, np.exp(rng.uniform(np.log(1e-4), 0, 512)), 1),
}
s = 1 + rng.pareto(1.5, 512)
cases["cfg5-like pareto"] = O.controlled_spectrum_matrix(2048, 512, 1e-6 + (s - s.min()) / (s.max() - s.min()), 2)
cases["gauss 4096x1024"] = rng.standard_normal((4096, 1024))
spec = U.MethodSpec(U.MethodKind.UNSO, coeffs=U.default_coefficients())
out = []
for name, m in cases.items():
    x = torch.from_numpy(m).to(torch.bfloat16).cuda()
    res = U.orthogonalize(x, spec, precision="bf16")
    ref = O.run(x.double().cpu().numpy(), "unso")["y"]
    err = np.linalg.norm(res.y.double().cpu().numpy() - ref) / np.linalg.norm(ref)
    out.append(f"{name}: {err:.2e} (steps {res.info[0]['chain_steps']:.0f})")
print(os.environ.get("UNSO_PCHAIN_HI_ONLY", "default"), " | ".join(out))
