"""CPU emulation of an Ozaki-style int8 split for the fp32 mode (dev tool, decides the slice counts).

A product A @ B is computed as exact int8 x int8 -> int32 slice products (tcgen05 kind::i8): every
row of A (column of B) is scaled by a power of two so its largest entry lies in [1/2, 1), then split
into S signed digits d_1 .. d_S with |d_s| <= 64 (first digit 6 bits, then 7 bits each, round to
nearest so the remainder keeps its sign freedom); the products with s + t <= S + 1 are summed
(triangle, S(S+1)/2 slice products; products with the same s + t share one int32 accumulator)
and rescaled in fp64.  Int8 products summed over K are exact in fp64 here (|sum| < 2^53), so the
emulation is exact.

usage: python tools/ozaki_emulation.py [cfg2|cfg5s|gauss] [S_gram S_chain S_apply]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import unso_oracle as O  # noqa: E402


def split_rows(a, S):
    """a (m x k) -> (exponents e (m,), digits list of S int-valued fp64 arrays): a = 2^e * sum d_s 2^-(6+7(s-1))."""
    mx = np.max(np.abs(a), axis=1)
    e = np.where(mx > 0, np.ceil(np.log2(np.where(mx > 0, mx, 1.0))), 0.0)
    r = a / np.exp2(e)[:, None]          # |r| <= 1
    digs = []
    r = r * 64.0
    for s in range(S):
        d = np.rint(r)
        digs.append(d)
        r = (r - d) * 128.0
    return e, digs


def ozaki(a, b, S):
    ea, da = split_rows(a, S)
    eb, db = split_rows(b.T, S)
    out = np.zeros((a.shape[0], b.shape[1]))
    for d in range(2, S + 2):           # s + t = d (1-based), triangle s + t <= S + 1
        acc = np.zeros_like(out)
        for s in range(1, d):
            t = d - s
            if s > S or t > S:
                continue
            acc += da[s - 1] @ db[t - 1].T   # exact int32 in hardware, exact here
        assert np.max(np.abs(acc)) < 2 ** 31, "int32 accumulator overflow"
        out += acc * 2.0 ** (-12 - 7 * (d - 2))
    return out * np.exp2(ea)[:, None] * np.exp2(eb)[None, :]


def unso_ozaki(m, Sg, Sc, Sa, order=14):
    x = np.asarray(m, np.float64)
    if x.shape[0] > x.shape[1]:
        x = x.T
    g = ozaki(x, x.T, Sg) if Sg else x @ x.T
    s = np.sqrt(np.sqrt(np.sum(g * g)))
    xs = x / s
    gs = g / (s * s)
    a = np.array(O.DEFAULT_A)
    b = O.final_coefficient(order, a, O.DEFAULT_RULE)
    h = gs.shape[0]
    # C-form: C_1 = G/s^2, C_{k+1} = 2 C_k - C_k^2; P = (1 + sum a + b) I - sum a_k C_k - b C_N
    co = list(a) + [b]
    C = gs
    P = (1.0 + sum(co)) * np.eye(h) - co[0] * C
    for k in range(1, order):
        sq = ozaki(C, C, Sc) if Sc else C @ C
        C = 2.0 * C - sq
        P = P - co[k] * C
    y = ozaki(P, xs, Sa) if Sa else P @ xs
    return y


def case(name):
    rng = np.random.default_rng(3)
    if name == "cfg2":
        s = np.exp(rng.uniform(np.log(1e-4), 0.0, 512))
        return O.controlled_spectrum_matrix(2048, 512, s, 11).astype(np.float32).astype(np.float64)
    if name == "cfg5s":
        s = rng.pareto(1.5, 512) + 1.0
        s = 1e-6 + (s - s.min()) / (s.max() - s.min()) * (1.0 - 1e-6)
        return O.controlled_spectrum_matrix(1024, 512, s, 12).astype(np.float32).astype(np.float64)
    return rng.standard_normal((2048, 512)).astype(np.float32).astype(np.float64)


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    m = case(name)
    ref = O.run(m, "unso")["y"]
    if ref.shape != m.shape:
        pass
    refT = ref if m.shape[0] <= m.shape[1] else ref.T
    combos = [tuple(int(v) for v in sys.argv[2:5])] if len(sys.argv) > 4 else \
        [(0, 0, 0), (4, 6, 5), (4, 5, 5), (3, 6, 5), (4, 6, 4), (4, 7, 5), (5, 7, 6)]
    for sg, sc, sa in combos:
        y = unso_ozaki(m, sg, sc, sa)
        err = np.linalg.norm(y - refT) / np.linalg.norm(refT)
        print(f"{name}: slices gram {sg} chain {sc} apply {sa}: rel err vs oracle {err:.2e}", flush=True)
