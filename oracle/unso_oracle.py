"""numpy float64 restatement of the UNSO reference hot path (TEST INFRASTRUCTURE ONLY).

See ``oracle/__init__.py`` for who may use this module.  All citations are
relative to ``/root/reference/pkg/src/unso/``.

Arithmetic follows the reference operation-for-operation (contiguous
transposes before products, the same axpy forms) so that results agree with
the live reference bit-for-bit on the same numpy/BLAS; the golden tests
allow 1e-12 to stay robust to a different BLAS on the GPU box host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "MUON_ABC", "DEFAULT_ORDER", "DEFAULT_RULE", "DEFAULT_A", "CESISTA_DEFAULT_TRIPLES",
    "stream_words", "stream_uniforms", "stream_normals", "gaussian_matrix",
    "final_coefficient", "poly_value", "constraint_point",
    "axpy_cost", "model_flops", "ContractionLog",
    "scale_and_orient", "unso_poly", "cubic_ns", "quintic_ns",
    "muon_rows", "cesista_rows", "run", "ortho_error", "ortho_error_any",
    "composed_map", "haar_columns", "controlled_spectrum_matrix", "unso_sampled", "quintic_sampled",
    "unso_rows_of_tall",
]

# ---------------------------------------------------------------------------
# constants restated from the reference
# ---------------------------------------------------------------------------

#: Muon quintic coefficients (ortho.py:49)
MUON_ABC = (3.4445, -4.7750, 2.0315)
#: default iteration counts (ortho.py:50-51)
ORIGINAL_DEFAULT_ITERS = 8
MUON_DEFAULT_ITERS = 5

#: shipped order-14 coefficient set, rule "exact" (data/default_coeffs.txt:1-14)
DEFAULT_ORDER = 14
DEFAULT_RULE = "exact"
DEFAULT_A = (
    0.50086411278516607, 0.43031295617574761, 0.85505919210311687,
    0.9411735833682553, 1.8241878615923741, 1.7434606137321689,
    3.8879837780264714, 3.4963822517823648, 5.91813134758823,
    16.085423985558819, -18.813955991531998, 106.33656092459489,
    -144.71993238023114,
)
#: shipped Cesista (gamma, r, l) schedule (data/cesista_default.txt:1-5)
CESISTA_DEFAULT_TRIPLES = (
    (2.1733754982919606, 0.2328021019681312, 0.38031317767627409),
    (2.6624433625932351, 0.55645800201365092, 0.27420893497388282),
    (1.912223714895789, 0.39404461123360224, 0.15186821763610917),
    (1.8549651820056539, 0.31103367329593429, 0.21232030281385791),
    (1.4745990163369547, 0.046492023078773308, -0.022323841840122156),
)

# ---------------------------------------------------------------------------
# counter-based PRNG: splitmix64 finalizer over a Weyl sequence (rng.py:18-61)
# ---------------------------------------------------------------------------

_U64 = np.uint64
_WEYL = _U64(0x9E3779B97F4A7C15)       # rng.py:18
_M1 = _U64(0xBF58476D1CE4E5B9)         # rng.py:19
_M2 = _U64(0x94D049BB133111EB)         # rng.py:20
_SALT = _U64(0x8E2B5CA19B3D71F7)       # rng.py:21


def _finalize64(z):
    """splitmix64 output mix (rng.py:24-28), modular uint64 arithmetic."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U64(30))) * _M1
        z = (z ^ (z >> _U64(27))) * _M2
        return z ^ (z >> _U64(31))


def stream_words(seed: int, start: int, count: int) -> np.ndarray:
    """uint64 words for counters start..start+count-1 (rng.py:31-40).

    Counter i (0-based) mixes base(seed) + (i+1)*golden; base is the mixed
    salted seed (rng.py:31-33)."""
    with np.errstate(over="ignore"):
        base = _finalize64(_U64(seed) + _SALT)
        ctr = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        return _finalize64(base + ctr * _WEYL)


def stream_uniforms(seed: int, start: int, count: int) -> np.ndarray:
    """Top 53 bits, centred in their cell -> strictly inside (0,1) (rng.py:43-46)."""
    w = stream_words(seed, start, count)
    return ((w >> _U64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def stream_normals(seed: int, start: int, count: int) -> np.ndarray:
    """Box-Muller over the first/second halves of 2*ceil(count/2) uniforms
    (rng.py:54-67): cos branch first, then sin branch."""
    half = (count + 1) // 2
    u = stream_uniforms(seed, start, 2 * half)
    radius = np.sqrt(-2.0 * np.log(u[:half]))
    angle = 2.0 * np.pi * u[half:]
    return np.concatenate([radius * np.cos(angle), radius * np.sin(angle)])[:count]


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """Row-major i.i.d. N(0,1) test matrix (bench.py:64-68)."""
    if rows < 1 or cols < 1:
        raise ValueError(f"dimensions must be positive, got {rows}x{cols}")
    return stream_normals(seed, 0, rows * cols).reshape(rows, cols)


# ---------------------------------------------------------------------------
# scalar polynomial / final coefficient (scalarpoly.py)
# ---------------------------------------------------------------------------

def constraint_point(order: int) -> float:
    """x_N = 1/sqrt(2^N + 1), where f is pinned to 1 (scalarpoly.py:101-103)."""
    return 1.0 / math.sqrt(2.0 ** order + 1.0)


def final_coefficient(order: int, a, rule: str = "exact") -> float:
    """The derived last coefficient b (``derive_b``, scalarpoly.py:117-127,
    with the exact-rule weights of ``_exact_b_parts`` scalarpoly.py:107-114)."""
    a = np.asarray(a, dtype=np.float64)
    if rule == "exact":
        t = 2.0 ** order
        r = t / (t + 1.0)
        weights = np.array([r ** (2.0 ** (k - 1)) for k in range(1, order)])
        amplification = (1.0 / r) ** (2.0 ** (order - 1))
        return float((math.sqrt(t + 1.0) - 1.0 - float(a @ weights)) * amplification)
    closed = math.exp(0.5) * (2.0 ** (order / 2.0) - 1.0)
    if rule == "approx-sum":
        return float(closed - float(np.sum(a)))
    if rule == "approx-abs":
        return float(closed - float(np.sum(np.abs(a))))
    raise ValueError(f"unknown b-rule {rule!r}")


def poly_value(order: int, a, rule: str, x):
    """f(x) = x + sum_k a_k x(1-x^2)^(2^(k-1)) + b x(1-x^2)^(2^(N-1))
    (``eval_f``, scalarpoly.py:130-138)."""
    b = final_coefficient(order, a, rule)
    acc = x * 1.0
    p = 1.0 - x * x
    for k in range(1, order):
        acc = acc + a[k - 1] * (x * p)
        p = p * p
    return acc + b * (x * p)


# ---------------------------------------------------------------------------
# FLOP model (densemat.py:33-51, 89-99; ortho.py:313-335)
# ---------------------------------------------------------------------------

def axpy_cost(alpha: float, beta: float, n: int) -> int:
    """1 op per non-unit scale and per add; beta==0 skips both (densemat.py:89-99)."""
    ops = n if alpha != 1.0 else 0
    if beta != 0.0:
        ops += n + (n if beta != 1.0 else 0)
    return ops


@dataclass
class ContractionLog:
    """FLOP total plus the (m,k,n) of every product (densemat.py:33-51)."""
    total: int = 0
    shapes: list = field(default_factory=list)

    def product(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        m, k = a.shape
        k2, n = b.shape
        if k != k2:
            raise ValueError(f"product shape mismatch ({m},{k})@({k2},{n})")
        self.shapes.append((m, k, n))
        self.total += 2 * m * k * n
        return a @ b

    def axpy(self, alpha: float, a: np.ndarray, beta: float, b: np.ndarray) -> np.ndarray:
        self.total += axpy_cost(alpha, beta, a.size)
        if beta == 0.0:
            return alpha * a if alpha != 1.0 else a.copy()
        return alpha * a + beta * b


def _T(a: np.ndarray) -> np.ndarray:
    """Contiguous transpose copy, as the reference does (densemat.py:85-86)."""
    return np.ascontiguousarray(a.T)


def muon_rows(iterations: int) -> np.ndarray:
    """Muon schedule: the fixed triple repeated (ortho.py:120-123, 234-237)."""
    return np.tile(np.array(MUON_ABC), (iterations, 1))


def cesista_rows(triples) -> np.ndarray:
    """(gamma, r, l) -> quintic (a, b, c) (``expand_cesista_rows`` ortho.py:240-247):
    p=(1+r)^2, q=(1-l)^2, a=1+gamma*p*q, b=-gamma*(p+q), c=gamma."""
    t = np.asarray(triples, dtype=np.float64)
    p = (1.0 + t[:, 1]) ** 2
    q = (1.0 - t[:, 2]) ** 2
    g = t[:, 0]
    return np.column_stack([1.0 + g * p * q, -g * (p + q), g])


def model_flops(method: str, h: int, w: int, *, order: int = DEFAULT_ORDER, a=DEFAULT_A,
                rule: str = DEFAULT_RULE, iterations: int | None = None, rows=None) -> int:
    """Closed-form kernel FLOPs (``kernel_model_flops`` ortho.py:313-335)."""
    hh = h * h
    if method == "unso":
        f = 2 * hh * w + axpy_cost(1.0, -1.0, hh) + (order - 1) * 2 * hh * h
        f += sum(axpy_cost(1.0, float(ak), hh) for ak in a)
        f += axpy_cost(1.0, final_coefficient(order, a, rule), hh)
        return f + 2 * hh * w
    if method == "original":
        it = ORIGINAL_DEFAULT_ITERS if iterations is None else iterations
        per = 4 * hh * w + axpy_cost(3.0, -1.0, hh) + axpy_cost(0.5, 0.0, h * w)
        return it * per
    if rows is None:
        rows = muon_rows(MUON_DEFAULT_ITERS if iterations is None else iterations)
    f = 0
    for ac, bc, cc in rows:
        f += 6 * hh * w + axpy_cost(float(ac), float(bc), h * w) + axpy_cost(1.0, float(cc), h * w)
    return f


# ---------------------------------------------------------------------------
# the pipeline (ortho.py)
# ---------------------------------------------------------------------------

def scale_and_orient(m: np.ndarray, scaling: str, log: ContractionLog | None = None,
                     gelfand_power: int = 2):
    """Row-wide orientation + spectral rescale (``preprocess`` ortho.py:140-168).

    Returns (x, was_transposed, denom)."""
    log = log if log is not None else ContractionLog()
    if not np.any(m):
        raise ValueError("degenerate: input matrix is identically zero")   # ortho.py:147-148
    transposed = m.shape[0] > m.shape[1]                                      # ortho.py:149
    a = _T(m) if transposed else m
    if scaling == "plain":                                                    # ortho.py:153-154
        log.total += 2 * a.size
        denom = float(np.sqrt(np.sum(a * a)))
    else:
        g = log.product(a, _T(a))                                             # ortho.py:156 / 159
        if scaling == "gram":
            log.total += 2 * g.size
            denom = float(np.sqrt(float(np.sqrt(np.sum(g * g)))))            # ortho.py:157
        elif scaling == "gelfand":
            p = g
            for _ in range(gelfand_power - 1):                                # ortho.py:160-162
                p = log.product(p, g)
            log.total += 2 * p.size
            denom = float(np.sqrt(np.sum(p * p))) ** (1.0 / (2.0 * gelfand_power))
        else:
            raise ValueError(f"unknown scaling {scaling!r}")
    if not np.isfinite(denom) or denom <= 0.0:                               # ortho.py:164-165
        raise ValueError("degenerate: scaling denominator is not a positive finite number")
    return log.axpy(1.0 / denom, a, 0.0, a), transposed, denom               # ortho.py:167


def unso_poly(x: np.ndarray, order: int = DEFAULT_ORDER, a=DEFAULT_A, rule: str = DEFAULT_RULE,
              log: ContractionLog | None = None) -> np.ndarray:
    """Y = P(X X^T) X with P = I + sum_k a_k B_k + b B_N, B_1 = I - XX^T,
    B_{k+1} = B_k^2 (``unso`` ortho.py:171-205)."""
    log = log if log is not None else ContractionLog()
    h, w = x.shape
    if h > w:
        raise ValueError(f"shape: kernel expects rows <= cols, got {h}x{w}")  # ortho.py:186-187
    b = final_coefficient(order, a, rule)                                     # ortho.py:197
    eye = np.eye(h)
    bk = log.axpy(1.0, eye, -1.0, log.product(x, _T(x)))                      # ortho.py:198-199
    p = np.eye(h)                                                             # ortho.py:200
    for k in range(1, order):                                                 # ortho.py:201-203
        p = log.axpy(1.0, p, float(a[k - 1]), bk)
        bk = log.product(bk, bk)
    p = log.axpy(1.0, p, b, bk)                                               # ortho.py:204
    return log.product(p, x)                                                  # ortho.py:205


def cubic_ns(x: np.ndarray, iterations: int, log: ContractionLog | None = None) -> np.ndarray:
    """X <- 0.5 (3I - XX^T) X (``original_ns`` ortho.py:208-218)."""
    log = log if log is not None else ContractionLog()
    h, w = x.shape
    if h > w:
        raise ValueError(f"shape: kernel expects rows <= cols, got {h}x{w}")
    eye = np.eye(h)
    for _ in range(iterations):
        lhs = log.axpy(3.0, eye, -1.0, log.product(x, _T(x)))
        x = log.axpy(0.5, log.product(lhs, x), 0.0, x)
    return x


def quintic_ns(x: np.ndarray, rows, log: ContractionLog | None = None) -> np.ndarray:
    """Per row (a,b,c): G=XX^T, p1=G X, p2=G p1, X = aX + b p1 + c p2
    (``_quintic_steps`` ortho.py:221-231)."""
    log = log if log is not None else ContractionLog()
    h, w = x.shape
    if h > w:
        raise ValueError(f"shape: kernel expects rows <= cols, got {h}x{w}")
    for ac, bc, cc in np.asarray(rows, dtype=np.float64):
        g = log.product(x, _T(x))
        p1 = log.product(g, x)
        p2 = log.product(g, p1)
        x = log.axpy(float(ac), x, float(bc), p1)
        x = log.axpy(1.0, x, float(cc), p2)
    return x


def _native_scaling(method: str) -> str:
    """UNSO defaults to gram scaling, the NS baselines to plain (ortho.py:112-118)."""
    return "gram" if method == "unso" else "plain"


def run(m: np.ndarray, method: str = "unso", *, scaling: str | None = None, order: int = DEFAULT_ORDER,
        a=DEFAULT_A, rule: str = DEFAULT_RULE, iterations: int | None = None, rows=None,
        gelfand_power: int = 2) -> dict:
    """preprocess -> kernel -> restore orientation (``orthogonalize`` ortho.py:259-283)."""
    m = np.asarray(m, dtype=np.float64)
    pre, ker = ContractionLog(), ContractionLog()
    x, transposed, denom = scale_and_orient(m, scaling or _native_scaling(method), pre, gelfand_power)
    if method == "unso":
        y = unso_poly(x, order, a, rule, ker)
    elif method == "original":
        y = cubic_ns(x, ORIGINAL_DEFAULT_ITERS if iterations is None else iterations, ker)
    else:
        if rows is None:
            rows = muon_rows(MUON_DEFAULT_ITERS if iterations is None else iterations)
        y = quintic_ns(x, rows, ker)
    if transposed:
        y = _T(y)
    return {"y": y, "flops": ker.total, "was_transposed": transposed,
            "preprocess_flops": pre.total, "shapes": ker.shapes, "denom": denom}


def ortho_error(y: np.ndarray) -> float:
    """||Y Y^T - I||_F for row-wide Y (bench.py:71-77)."""
    h, w = y.shape
    if h > w:
        raise ValueError(f"shape: ortho_error expects rows <= cols, got {h}x{w}")
    return float(np.linalg.norm(y @ y.T - np.eye(h)))


def ortho_error_any(y: np.ndarray) -> float:
    """Short-side orientation first (bench.py:80-82)."""
    return ortho_error(y if y.shape[0] <= y.shape[1] else _T(y))


def composed_map(method: str, *, order: int = DEFAULT_ORDER, a=DEFAULT_A, rule: str = DEFAULT_RULE,
                 iterations: int | None = None, rows=None):
    """Scalar map applied to each singular value (``scalar_map`` ortho.py:286-310)."""
    if method == "unso":
        return lambda s: poly_value(order, a, rule, s)
    if method == "original":
        it = ORIGINAL_DEFAULT_ITERS if iterations is None else iterations

        def cubic(s):
            y = np.asarray(s, dtype=np.float64) * 1.0
            for _ in range(it):
                y = 0.5 * y * (3.0 - y * y)
            return y
        return cubic
    if rows is None:
        rows = muon_rows(MUON_DEFAULT_ITERS if iterations is None else iterations)
    rows = np.asarray(rows, dtype=np.float64)

    def quintic(s):
        y = np.asarray(s, dtype=np.float64) * 1.0
        for ac, bc, cc in rows:
            yy = y * y
            y = y * (ac + bc * yy + cc * yy * yy)
        return y
    return quintic


def unso_rows_of_tall(m: np.ndarray, rows: np.ndarray, order: int = DEFAULT_ORDER, a=DEFAULT_A,
                      rule: str = DEFAULT_RULE) -> np.ndarray:
    """Selected rows of orthogonalize(m) for a tall m (w x h, w > h), computed with the
    reference's operations (ortho.py:140-205) but applying P only to the requested rows:
    (P X^T)^T restricted to `rows` = X[rows] P (P symmetric).  For full-size parity
    checks where forming all of Y on the host is unnecessary."""
    x = np.ascontiguousarray(m.T)                               # preprocess transposes (ortho.py:149-150)
    g = x @ _T(x)                                               # ortho.py:156
    denom = float(np.sqrt(float(np.sqrt(np.sum(g * g)))))       # ortho.py:157
    g = g / (denom * denom)                                     # == (x/denom)(x/denom)^T up to rounding
    b = final_coefficient(order, a, rule)
    h = g.shape[0]
    bk = np.eye(h) - g
    p = np.eye(h)
    for k in range(1, order):
        p = p + float(a[k - 1]) * bk
        bk = bk @ bk
    p = p + b * bk
    return (m[rows] / denom) @ p



def _oriented(m: np.ndarray):
    """Row-wide orientation of preprocess (ortho.py:149-150): transpose iff rows > cols."""
    tall = m.shape[0] > m.shape[1]
    return (np.ascontiguousarray(m.T) if tall else np.asarray(m, dtype=np.float64)), tall


def unso_sampled(m: np.ndarray, idx, order: int = DEFAULT_ORDER, a=DEFAULT_A, rule: str = DEFAULT_RULE,
                 scaling: str = "gram") -> np.ndarray:
    """orthogonalize(m, UNSO) restricted to long-side indices `idx`, any orientation: rows idx of
    Y for a tall m, columns idx of Y for a wide or square m.  Same operations as the reference
    (ortho.py:140-205): gram / plain scale (:153-157), B_1 = I - G (:199), P += a_k B_k,
    B <- B B (:201-203), P += b B_N (:204), Y = P X (:205) -- with P applied only to the requested
    long-side columns of X (each column of P X depends on that column of X alone).  For
    full-size parity checks of BASELINE configs[2]-[4] where forming all of Y is unnecessary."""
    x, tall = _oriented(m)
    g = x @ _T(x)                                               # ortho.py:156 (the Gram of A)
    if scaling == "gram":
        denom = float(np.sqrt(float(np.sqrt(np.sum(g * g)))))   # ortho.py:157
    elif scaling == "plain":
        denom = float(np.sqrt(float(np.sum(x * x))))             # ortho.py:153-154
    else:
        raise ValueError("unso_sampled supports gram and plain scaling")
    g = g / (denom * denom)                                     # == (x/denom)(x/denom)^T up to rounding
    b = final_coefficient(order, a, rule)
    h = g.shape[0]
    bk = np.eye(h) - g
    p = np.eye(h)
    for k in range(1, order):
        p = p + float(a[k - 1]) * bk
        bk = bk @ bk
    p = p + b * bk
    y = p @ (x[:, idx] / denom)                                 # columns idx of P X
    return np.ascontiguousarray(y.T) if tall else y


def quintic_sampled(m: np.ndarray, idx, rows=None) -> np.ndarray:
    """The quintic NS iteration (_quintic_steps ortho.py:221-231 after plain scaling, :153-154)
    restricted to long-side indices `idx` (rows of Y if tall, else columns).  Every iterate is
    X_k = M_k X_0 with M_k a polynomial in G_0 = X_0 X_0^T, so G_k = M_k G_0 M_k and
    M_{k+1} = (a I + b G_k + c G_k^2) M_k: the same map in h x h arithmetic (exact restatement;
    pinned against quintic_ns on small cases by tests/test_oracle_golden.py), then Y = M_T X_0."""
    if rows is None:
        rows = muon_rows(MUON_DEFAULT_ITERS)
    x, tall = _oriented(m)
    x = x / float(np.sqrt(float(np.sum(x * x))))
    g0 = x @ _T(x)
    h = g0.shape[0]
    mk = np.eye(h)
    for ac, bc, cc in np.asarray(rows, dtype=np.float64):
        gk = mk @ g0 @ mk
        mk = (float(ac) * np.eye(h) + float(bc) * gk + float(cc) * (gk @ gk)) @ mk
    y = mk @ x[:, idx]
    return np.ascontiguousarray(y.T) if tall else y


# ---------------------------------------------------------------------------
# controlled-spectrum inputs (BASELINE.json configs[1], configs[4])
# ---------------------------------------------------------------------------

def haar_columns(n: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """First k columns of a Haar-random n x n orthogonal matrix: QR of a
    Gaussian n x k with the sign fix diag(R) > 0."""
    q, r = np.linalg.qr(rng.standard_normal((n, k)))
    return q * np.sign(np.diag(r))


def controlled_spectrum_matrix(rows: int, cols: int, s: np.ndarray, seed: int) -> np.ndarray:
    """X = U diag(s) V^T with U (rows x k), V (cols x k) Haar, k=min(rows,cols)."""
    rng = np.random.default_rng(seed)
    k = min(rows, cols)
    u = haar_columns(rows, k, rng)
    v = haar_columns(cols, k, rng)
    return (u * s[None, :]) @ v.T
