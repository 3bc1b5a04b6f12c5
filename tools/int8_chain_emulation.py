"""Dev tool: the bf16-mode large-h chain with int8 digit products (S digits, triangle of products)
instead of bf16 hi*hi + e4m3 cross terms -- precision of the whole UNSO result against the oracle on
the BASELINE-like spectra (apply exact, so the chain error is isolated).  S=2: 3 int8 products =
1.5 bf16-equivalents of tensor time per squaring, vs 2 for the shipped recipe."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import unso_oracle as O  # noqa: E402
from tools.ozaki_emulation import ozaki  # noqa: E402


def rnd_bits(a, drop):
    u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    half = (1 << (drop - 1)) - 1
    u = ((u + half + ((u >> drop) & 1)) >> drop) << drop
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


bf16 = lambda a: rnd_bits(a, 16)


def chain(m, S, first_bf16_hi=0):
    x = np.asarray(m, np.float64)
    if x.shape[0] > x.shape[1]:
        x = x.T
    g = x @ x.T
    s2 = np.sqrt(np.sum(g * g))
    C = (g / s2).astype(np.float32).astype(np.float64)
    a = np.array(O.DEFAULT_A)
    co = list(a) + [O.final_coefficient(14, a, "exact")]
    P = (1 + sum(co)) * np.eye(C.shape[0]) - co[0] * C
    for k in range(1, 14):
        if k <= first_bf16_hi:
            h = bf16(C)
            sq = h @ h
        else:
            sq = ozaki(C, C, S)
        C = (2 * C - sq).astype(np.float32).astype(np.float64)
        P = P - co[k] * C
    return (P / np.sqrt(s2)) @ x


rng = np.random.default_rng(0)
cases = {
    "cfg3-like 1024^2 N(0,.02^2)": bf16(rng.standard_normal((1024, 1024)) * 0.02),
    "cfg3-like tall 3584x1024": bf16(rng.standard_normal((3584, 1024)) * 0.02),
    "cfg2-like 2048x512 logU[1e-4,1]": bf16(O.controlled_spectrum_matrix(2048, 512, np.exp(rng.uniform(np.log(1e-4), 0, 512)), 1)),
}
s = 1 + rng.pareto(1.5, 512)
s = 1e-6 + (s - s.min()) / (s.max() - s.min()) * (1 - 1e-6)
cases["cfg5-like 2048x512 pareto"] = bf16(O.controlled_spectrum_matrix(2048, 512, s, 2))
for name, m in cases.items():
    ref = O.run(m, "unso")["y"]
    ref = ref if ref.shape[0] <= ref.shape[1] else ref.T
    out = []
    for S, first in ((2, 0), (2, 3), (3, 0)):
        y = chain(m, S, first)
        out.append(f"S={S},hi-first{first}={np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}")
    print(name, " ".join(out), flush=True)
