"""CPU emulation of squaring-chain precision recipes (operand rounding emulated exactly,
products/accumulation in fp64).  Dev tool used to choose the chain recipe; see DESIGN.md."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import unso_oracle as O

def rnd_bits(a, drop):
    u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    half = (1 << (drop - 1)) - 1
    u = ((u + half + ((u >> drop) & 1)) >> drop) << drop
    return u.astype(np.uint32).view(np.float32).astype(np.float64)
bf16 = lambda a: rnd_bits(a, 16)
tf32 = lambda a: rnd_bits(a, 13)
def e4m3(a):  # 3 mantissa bits, normal range only (inputs pre-scaled into range)
    a = np.asarray(a, np.float64); m, e = np.frexp(a)
    return np.ldexp(np.round(m * 16) / 16, e)

def chain(C, mode):
    def sq(C):
        if mode == "fp64": return C @ C
        if mode == "bf16x3":
            h = bf16(C); l = bf16(C - h); return h @ h + h @ l + l @ h
        if mode == "tf32": t = tf32(C); return t @ t
        if mode == "tf32x2":  # t*t + t*l + l*t  with tf32 split
            t = tf32(C); l = tf32(C - t); return t @ t + t @ l + l @ t
        if mode == "bf16+fp8x":
            h = bf16(C); l = C - h
            h8 = e4m3(h); l8 = e4m3(l * 256.0) / 256.0
            return h @ h + h8 @ l8 + l8 @ h8
        raise ValueError(mode)
    return sq

def unso_cform(m, mode, bf_input=True):
    x = np.asarray(m, np.float64)
    if x.shape[0] > x.shape[1]: x = x.T
    g = x @ x.T; s2 = np.sqrt(np.sum(g * g)); C = (g / s2).astype(np.float32).astype(np.float64)
    a = np.array(O.DEFAULT_A); c = O.final_coefficient(14, a, "exact"); co = list(a) + [c]
    sq = chain(C, mode); alpha = 1 + sum(co)
    P = alpha * np.eye(C.shape[0]) - co[0] * C
    for k in range(1, 14):
        C = (2 * C - sq(C)).astype(np.float32).astype(np.float64)
        P = P - co[k] * C
    return (P / np.sqrt(s2)) @ x   # exact apply: isolate chain error

rng = np.random.default_rng(0)
cases = {
  "cfg3-like 1024^2 N(0,.02^2)": bf16(rng.standard_normal((1024, 1024)) * 0.02),
  "cfg3-like tall 3584x1024": bf16(rng.standard_normal((3584, 1024)) * 0.02),
  "cfg2-like 2048x512 logU[1e-4,1]": bf16(O.controlled_spectrum_matrix(2048, 512, np.exp(rng.uniform(np.log(1e-4), 0, 512)), 1)),
}
s = 1 + rng.pareto(1.5, 512); s = 1e-6 + (s - s.min()) / (s.max() - s.min()) * (1 - 1e-6)
cases["cfg5-like 2048x512 pareto"] = bf16(O.controlled_spectrum_matrix(2048, 512, s, 2))
for name, m in cases.items():
    ref = O.run(m, "unso")["y"]; ref = ref if ref.shape[0] <= ref.shape[1] else ref.T
    out = []
    for mode in ("fp64", "bf16x3", "tf32x2", "bf16+fp8x", "tf32"):
        y = unso_cform(m, mode)
        out.append(f"{mode}={np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}")
    print(name, " ".join(out), flush=True)


def e4m3_real(a):
    """e4m3 with range: max 448, subnormals spaced 2^-9 below 2^-6, RNE."""
    a = np.asarray(a, np.float64)
    sgn = np.sign(a); x = np.abs(a)
    e = np.floor(np.log2(np.maximum(x, 1e-300)))
    e = np.maximum(e, -6)                      # subnormal region uses exponent -6
    q = np.ldexp(1.0, (e - 3).astype(int))     # spacing: 3 mantissa bits
    r = np.round(x / q) * q
    return sgn * np.minimum(r, 448.0)


def chain_fp8_scaled(C, S_hi=8, S_lo=16):
    h = bf16(C); l = C - h
    h8 = e4m3_real(h * 2.0 ** S_hi) / 2.0 ** S_hi
    l8 = e4m3_real(l * 2.0 ** S_lo) / 2.0 ** S_lo
    return h @ h + h8 @ l8 + l8 @ h8


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "fp8":
    for name, m in cases.items():
        ref = O.run(m, "unso")["y"]; ref = ref if ref.shape[0] <= ref.shape[1] else ref.T
        for S_hi, S_lo in ((8, 16), (8, 17), (7, 15)):
            x = np.asarray(m, np.float64); x = x.T if x.shape[0] > x.shape[1] else x
            g = x @ x.T; s2 = np.sqrt(np.sum(g * g)); C = (g / s2).astype(np.float32).astype(np.float64)
            a = np.array(O.DEFAULT_A); c = O.final_coefficient(14, a, "exact"); co = list(a) + [c]
            P = (1 + sum(co)) * np.eye(C.shape[0]) - co[0] * C
            for k in range(1, 14):
                C = (2 * C - chain_fp8_scaled(C, S_hi, S_lo)).astype(np.float32).astype(np.float64)
                P = P - co[k] * C
            y = (P / np.sqrt(s2)) @ x
            print(name, f"S=({S_hi},{S_lo})", f"{np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}", flush=True)


def unso_first_steps_hi_only(m, first, bf16x3=False):
    """The large-h recipe (bf16 hi*hi + e4m3 cross terms; C_k stored as bf16 hi + bf16 lo) with the
    cross terms dropped in the first `first` squarings (bf16x3=True: the bf16x3 recipe instead)."""
    x = np.asarray(m, np.float64)
    if x.shape[0] > x.shape[1]: x = x.T
    g = x @ x.T; s2 = np.sqrt(np.sum(g * g)); C = (g / s2).astype(np.float32).astype(np.float64)
    a = np.array(O.DEFAULT_A); c = O.final_coefficient(14, a, "exact"); co = list(a) + [c]
    P = (1 + sum(co)) * np.eye(C.shape[0]) - co[0] * C
    for k in range(1, 14):
        h = bf16(C)
        if bf16x3:
            l = bf16(C - h)
            sq = h @ h if k <= first else h @ h + h @ l + l @ h
            n = 2 * C - sq
        else:
            l = C - h
            if k <= first:
                sq = h @ h
            else:
                h8 = e4m3_real(h * 256.0) / 256.0; l8 = e4m3_real(l * 65536.0) / 65536.0
                sq = h @ h + h8 @ l8 + l8 @ h8
            n = 2 * (h + bf16(l)) - sq
        C = n.astype(np.float32).astype(np.float64)
        P = P - co[k] * C
    return (P / np.sqrt(s2)) @ x


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--first-steps":
    # cross terms dropped in the first j squarings (what the large-h chain ships with j = 2)
    for name, m in cases.items():
        ref = O.run(m, "unso")["y"]; ref = ref if ref.shape[0] <= ref.shape[1] else ref.T
        r = {f"first{j}": np.linalg.norm(unso_first_steps_hi_only(m, j) - ref) / np.linalg.norm(ref)
             for j in (0, 1, 2, 3, 4)}
        print(name, " ".join(f"{k}={v:.2e}" for k, v in r.items()), flush=True)
