"""Host-side coefficient handling for the UNSO polynomial.

Mirrors the reference's ``unso.scalarpoly`` entry points that the hot path
needs (scalarpoly.py:31-61, 101-138, 181-218):

    f(x) = x + sum_{k=1}^{N-1} a_k x (1-x^2)^(2^(k-1)) + b x (1-x^2)^(2^(N-1))

``derive_b`` solves for the last coefficient from the pin f(1/sqrt(2^N+1)) = 1.
These are O(N) scalar computations done once per coefficient set on the host;
the matrix work happens in the CUDA library.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from enum import Enum
from importlib import resources

import numpy as np

from .errors import ParseError


class BRule(str, Enum):
    """How the final coefficient is derived (scalarpoly.py:31-36)."""

    EXACT = "exact"
    APPROX_SUM = "approx-sum"
    APPROX_ABS = "approx-abs"


@dataclass(frozen=True)
class CoefficientSet:
    """Order-N coefficients: N-1 learnable a_k plus the rule for b (scalarpoly.py:39-61)."""

    order: int
    a: np.ndarray = field(default=None)  # type: ignore[assignment]
    b_rule: BRule = BRule.EXACT

    def __post_init__(self):
        if self.order < 1:
            raise ValueError(f"order must be >= 1, got {self.order}")
        a = np.zeros(self.order - 1) if self.a is None else np.array(self.a, dtype=np.float64)
        if a.shape != (self.order - 1,):
            raise ValueError(f"expected {self.order - 1} learnable coefficients, got {a.shape}")
        if not np.all(np.isfinite(a)):
            raise ValueError("coefficients must be finite")
        a.setflags(write=False)
        object.__setattr__(self, "a", a)
        object.__setattr__(self, "b_rule", BRule(self.b_rule))

    def with_a(self, a) -> "CoefficientSet":
        return CoefficientSet(self.order, a, self.b_rule)

    def device_coefficients(self) -> np.ndarray:
        """The N values the C ABI takes: a_1..a_{N-1}, then b."""
        return np.concatenate([self.a, [derive_b(self)]]).astype(np.float64)


def constraint_point(order: int) -> float:
    """x_N = 1/sqrt(2^N + 1), the peak of the last term (scalarpoly.py:101-103)."""
    return 1.0 / math.sqrt(2.0 ** order + 1.0)


def derive_b(coeffs: CoefficientSet) -> float:
    """Final coefficient under the set's rule (scalarpoly.py:117-127).

    exact:      b = (sqrt(2^N+1) - 1 - sum_k a_k r^(2^(k-1))) / r^(2^(N-1)),  r = 2^N/(2^N+1)
    approx-sum: b = e^(1/2) (2^(N/2) - 1) - sum a_k
    approx-abs: b = e^(1/2) (2^(N/2) - 1) - sum |a_k|
    """
    n = coeffs.order
    if coeffs.b_rule is BRule.EXACT:
        t = 2.0 ** n
        r = t / (t + 1.0)
        q = np.array([r ** (2.0 ** (k - 1)) for k in range(1, n)])
        inv_last = (1.0 / r) ** (2.0 ** (n - 1))
        return float((math.sqrt(t + 1.0) - 1.0 - float(coeffs.a @ q)) * inv_last)
    base = math.exp(0.5) * (2.0 ** (n / 2.0) - 1.0)
    if coeffs.b_rule is BRule.APPROX_SUM:
        return float(base - float(np.sum(coeffs.a)))
    return float(base - float(np.sum(np.abs(coeffs.a))))


def eval_f(coeffs: CoefficientSet, x):
    """f at scalar/array x via repeated squaring of (1-x^2) (scalarpoly.py:130-138)."""
    b = derive_b(coeffs)
    x = np.asarray(x, dtype=np.float64) if not np.isscalar(x) else float(x)
    acc = x * 1.0
    p = 1.0 - x * x
    for k in range(1, coeffs.order):
        acc = acc + coeffs.a[k - 1] * (x * p)
        p = p * p
    return acc + b * (x * p)


def constraint_residual(coeffs: CoefficientSet) -> float:
    """f(x_N) - 1; zero up to rounding under the exact rule (scalarpoly.py:141-143)."""
    return float(eval_f(coeffs, constraint_point(coeffs.order))) - 1.0


def write_coefficients(path, coeffs: CoefficientSet) -> None:
    """The reference's text format: "<N> <rule>" then one a_k per line (scalarpoly.py:181-189)."""
    lines = [f"{coeffs.order} {coeffs.b_rule.value}"] + [f"{v:.17g}" for v in coeffs.a]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def read_coefficients(path) -> CoefficientSet:
    """Parse the reference's coefficient text format (scalarpoly.py:192-218)."""
    with open(path) as fh:
        lines = [ln.strip() for ln in fh.read().split("\n") if ln.strip()]
    if not lines:
        raise ParseError(f"{path}: empty coefficient file")
    head = lines[0].split()
    if len(head) != 2:
        raise ParseError(f"{path}: header must be '<order> <b-rule>'")
    try:
        order = int(head[0])
    except ValueError as exc:
        raise ParseError(f"{path}: non-integer order") from exc
    try:
        rule = BRule(head[1])
    except ValueError as exc:
        raise ParseError(f"{path}: unknown b-rule {head[1]!r}") from exc
    if len(lines) - 1 != order - 1:
        raise ParseError(f"{path}: expected {order - 1} coefficients, found {len(lines) - 1}")
    try:
        a = np.array([float(v) for v in lines[1:]], dtype=np.float64)
    except ValueError as exc:
        raise ParseError(f"{path}: non-numeric coefficient") from exc
    try:
        return CoefficientSet(order, a, rule)
    except ValueError as exc:
        raise ParseError(f"{path}: {exc}") from exc


def _load_json(name: str) -> dict:
    return json.loads(resources.files(__package__).joinpath("data", name).read_text())


def default_coefficients() -> CoefficientSet:
    """The shipped order-14 learned coefficients (reference data/__init__.py:24-25)."""
    d = _load_json("unso_default_order14.json")
    return CoefficientSet(int(d["order"]), np.array(d["a"], dtype=np.float64), BRule(d["b_rule"]))


@dataclass(frozen=True)
class CesistaStepParams:
    """Per-step (gamma, r, l) triples (reference coeff_train.py:68-86)."""

    triples: np.ndarray

    def __post_init__(self):
        t = np.array(self.triples, dtype=np.float64)
        if t.ndim != 2 or t.shape[1] != 3 or t.shape[0] < 1:
            raise ValueError(f"expected a (T, 3) array with T >= 1, got {t.shape}")
        if not np.all(np.isfinite(t)):
            raise ValueError("step parameters must be finite")
        t.setflags(write=False)
        object.__setattr__(self, "triples", t)

    @property
    def steps(self) -> int:
        return self.triples.shape[0]


def read_step_triples(path) -> np.ndarray:
    """Whitespace-separated 3-column schedule file (reference coeff_train.py:239-256)."""
    with open(path) as fh:
        lines = [ln.strip() for ln in fh.read().split("\n") if ln.strip()]
    if not lines:
        raise ParseError(f"{path}: empty schedule file")
    rows = []
    for i, line in enumerate(lines):
        parts = line.split()
        if len(parts) != 3:
            raise ParseError(f"{path}: line {i + 1} must hold exactly 3 values")
        try:
            rows.append([float(p) for p in parts])
        except ValueError as exc:
            raise ParseError(f"{path}: line {i + 1} has a non-numeric value") from exc
    out = np.array(rows, dtype=np.float64)
    if not np.all(np.isfinite(out)):
        raise ParseError(f"{path}: schedule contains non-finite values")
    return out


def default_cesista_triples() -> np.ndarray:
    """The shipped 5-step Cesista schedule (reference data/__init__.py:28-29)."""
    return np.array(_load_json("cesista_default_5step.json")["triples"], dtype=np.float64)
