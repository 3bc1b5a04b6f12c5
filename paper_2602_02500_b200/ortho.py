"""Orthogonalizers on B200: the reference's ``unso.ortho`` API over CUDA tensors.

Same entry points, argument meaning and exceptions as the reference
(``/root/reference/pkg/src/unso/ortho.py``):

    orthogonalize(m, spec) -> OrthoResult            ortho.py:267-283
    preprocess(m, scaling, counter, gelfand_power)   ortho.py:140-168
    unso(x, coeffs, counter, debug)                  ortho.py:171-205
    original_ns / muon_ns / cesista_ns               ortho.py:208-256
    kernel_model_flops(h, w, spec), scalar_map(spec) ortho.py:286-335

Inputs are CUDA tensors (float32 / bfloat16 / float64), 2-D or a 3-D batch of
equally shaped matrices; outputs have the input's shape and dtype.  All matrix
arithmetic runs in ``libunso_b200.so`` (hand-written sm_100a kernels, see
DESIGN.md); this module only validates, lays out descriptors and maps errors.

Added keywords (not in the reference): ``precision`` ("fp32": fp64-grade
internals, parity <= 1e-5; "bf16": tcgen05 tensor cores, parity <= 2e-2;
default: "bf16" for bfloat16 input, else "fp32"), ``check`` (read the device
status word and raise ``DegenerateInputError``; costs one host sync) and
``out`` (preallocated result).
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .errors import DegenerateInputError, ShapeError
from .scalarpoly import CesistaStepParams, CoefficientSet, derive_b, eval_f

MUON_COEFFICIENTS = (3.4445, -4.7750, 2.0315)      # ortho.py:49
DEFAULT_ORIGINAL_ITERATIONS = 8                    # ortho.py:50
DEFAULT_MUON_ITERATIONS = 5                        # ortho.py:51


class Scaling(str, Enum):
    """ortho.py:54-57"""
    FROBENIUS_GRAM = "gram"
    FROBENIUS_PLAIN = "plain"
    GELFAND = "gelfand"


class MethodKind(str, Enum):
    """ortho.py:60-65"""
    UNSO = "unso"
    ORIGINAL_NS = "original"
    MUON_NS = "muon"
    CESISTA_NS = "cesista"
    EXTERNAL_SCHEDULE = "external"


class Precision(str, Enum):
    """Arithmetic recipe (include/unso_b200.h)."""
    FP32 = "fp32"
    BF16 = "bf16"


@dataclass(frozen=True)
class MethodSpec:
    """A fully parameterised method (ortho.py:68-128), plus the device recipe."""

    kind: MethodKind
    iterations: int | None = None
    coeffs: CoefficientSet | None = None
    step_params: CesistaStepParams | None = None
    schedule: np.ndarray | None = None
    scaling: Scaling | None = None
    gelfand_power: int = 2
    precision: Precision | None = None
    apply_terms: int | None = None   # bf16 mode: None = adaptive per matrix, 1 = P_hi only, 2 = P_hi + P_lo
    chain: str | None = None         # bf16 mode, large h: None = bf16 hi*hi (first 3 squarings alone) + e4m3 cross terms, "bf16x3"
    truncate: bool = True            # bf16 mode, persistent chain: stop once ||I - C_k||_F bounds the rest
    ns_products: str | None = None   # bf16 mode, NS kinds: None / "bf16x3" = hi/lo state in the long-side
                                     # products (~1e-4 from fp64), "bf16" = one bf16 term (faster, ~1e-2)
    fp32_engine: str | None = None   # fp32 mode, UNSO, h > 256: None / "int8" = int8 tensor-core digit split
                                     # (~1e-7 from fp64), "dmma" = the fp64 tensor cores (~1e-14, slower)

    def __post_init__(self):
        object.__setattr__(self, "_cache", {})  # per-spec memo of the native method descriptor / FLOP model
        kind = MethodKind(self.kind)
        object.__setattr__(self, "kind", kind)
        if self.scaling is not None:
            object.__setattr__(self, "scaling", Scaling(self.scaling))
        if self.precision is not None:
            object.__setattr__(self, "precision", Precision(self.precision))
        if self.gelfand_power < 1:
            raise ValueError("gelfand_power must be >= 1")
        if self.apply_terms not in (None, 1, 2):
            raise ValueError("apply_terms must be None (adaptive), 1 or 2")
        if self.chain not in (None, "bf16x3"):
            raise ValueError("chain must be None (bf16 + e4m3 cross terms) or 'bf16x3'")
        if self.ns_products not in (None, "bf16x3", "bf16"):
            raise ValueError("ns_products must be None / 'bf16x3' (hi/lo state) or 'bf16'")
        if self.fp32_engine not in (None, "int8", "dmma"):
            raise ValueError("fp32_engine must be None / 'int8' (int8 tensor-core split) or 'dmma' (fp64)")
        if kind is MethodKind.UNSO:
            if self.coeffs is None:
                raise ValueError("unso requires a CoefficientSet")
        elif kind in (MethodKind.ORIGINAL_NS, MethodKind.MUON_NS):
            its = self.iterations
            if its is None:
                its = DEFAULT_ORIGINAL_ITERATIONS if kind is MethodKind.ORIGINAL_NS else DEFAULT_MUON_ITERATIONS
                object.__setattr__(self, "iterations", its)
            if its < 1:
                raise ValueError("iterative methods need iterations >= 1")
        elif kind is MethodKind.CESISTA_NS:
            if self.step_params is None:
                raise ValueError("cesista requires CesistaStepParams")
        else:
            sched = None if self.schedule is None else np.array(self.schedule, dtype=np.float64)
            if sched is None or sched.ndim != 2 or sched.shape[1] != 3 or sched.shape[0] < 1:
                raise ValueError("external schedule requires a (T, 3) coefficient array")
            sched.setflags(write=False)
            object.__setattr__(self, "schedule", sched)

    @property
    def effective_scaling(self) -> Scaling:
        """UNSO defaults to gram scaling, the NS baselines to plain (ortho.py:112-118)."""
        if self.scaling is not None:
            return self.scaling
        return Scaling.FROBENIUS_GRAM if self.kind is MethodKind.UNSO else Scaling.FROBENIUS_PLAIN

    def quintic_rows(self) -> np.ndarray:
        """Per-step (a, b, c) rows of the quintic kinds (ortho.py:120-128)."""
        if self.kind is MethodKind.MUON_NS:
            return np.tile(np.array(MUON_COEFFICIENTS), (self.iterations, 1))
        if self.kind is MethodKind.CESISTA_NS:
            return expand_cesista_rows(self.step_params.triples)
        if self.kind is MethodKind.EXTERNAL_SCHEDULE:
            return np.asarray(self.schedule, dtype=np.float64)
        raise ValueError(f"{self.kind.value} has no quintic schedule")


@dataclass
class OrthoResult:
    """ortho.py:131-137, plus what the device actually executed."""

    y: torch.Tensor
    flops: int                       # reference kernel-model FLOPs per matrix (excludes preprocessing)
    was_transposed: bool
    preprocess_flops: int = 0
    kernel_matmul_shapes: list[tuple[int, int, int]] = field(default_factory=list)
    executed_matmul_shapes: list[tuple[int, int, int]] = field(default_factory=list)
    precision: str = "fp32"
    launches: int = 0
    info: dict | None = None         # per-matrix device scalars (scale, apply decision, bound) when check=True


class FlopsCounter:
    """Reference-compatible FLOP accumulator (densemat.py:33-51)."""

    def __init__(self):
        self.total = 0
        self.matmul_shapes: list[tuple[int, int, int]] = []

    def add(self, count: int) -> None:
        if count < 0:
            raise ValueError(f"negative FLOPs increment: {count}")
        self.total += int(count)

    def record_matmul(self, m: int, k: int, n: int) -> None:
        self.matmul_shapes.append((m, k, n))
        self.add(2 * m * k * n)

    def reset(self) -> None:
        self.total = 0
        self.matmul_shapes.clear()


# ---------------------------------------------------------------------------- FLOP model

def _axpy_cost(alpha: float, beta: float, n: int) -> int:
    """densemat.py:89-99"""
    cost = n if alpha != 1.0 else 0
    if beta != 0.0:
        cost += n + (n if beta != 1.0 else 0)
    return cost


def kernel_model_flops(h: int, w: int, spec: MethodSpec) -> int:
    """Closed-form kernel FLOPs of the reference (ortho.py:313-335)."""
    hh = h * h
    if spec.kind is MethodKind.UNSO:
        c = spec.coeffs
        total = 2 * hh * w + _axpy_cost(1.0, -1.0, hh) + (c.order - 1) * 2 * hh * h
        total += sum(_axpy_cost(1.0, float(a), hh) for a in c.a)
        total += _axpy_cost(1.0, derive_b(c), hh) + 2 * hh * w
        return total
    if spec.kind is MethodKind.ORIGINAL_NS:
        per = 4 * hh * w + _axpy_cost(3.0, -1.0, hh) + _axpy_cost(0.5, 0.0, h * w)
        return spec.iterations * per
    total = 0
    for a, b, c in spec.quintic_rows():
        total += 6 * hh * w + _axpy_cost(float(a), float(b), h * w) + _axpy_cost(1.0, float(c), h * w)
    return total


def preprocess_model_flops(h: int, w: int, scaling: Scaling, gelfand_power: int = 2) -> int:
    """FLOPs the reference's preprocess charges (ortho.py:153-167)."""
    scaling = Scaling(scaling)
    if scaling is Scaling.FROBENIUS_PLAIN:
        return 2 * h * w + h * w
    if scaling is Scaling.FROBENIUS_GRAM:
        return 2 * h * h * w + 2 * h * h + h * w
    return 2 * h * h * w + (gelfand_power - 1) * 2 * h * h * h + 2 * h * h + h * w


def model_matmul_shapes(h: int, w: int, spec: MethodSpec) -> list[tuple[int, int, int]]:
    """The (m, k, n) audit the reference's counter records (densemat.py:45-47)."""
    if spec.kind is MethodKind.UNSO:
        return [(h, w, h)] + [(h, h, h)] * (spec.coeffs.order - 1) + [(h, h, w)]
    if spec.kind is MethodKind.ORIGINAL_NS:
        return [(h, w, h), (h, h, w)] * spec.iterations
    return [(h, w, h), (h, h, w), (h, h, w)] * len(spec.quintic_rows())


def executed_matmul_shapes(h: int, w: int, spec: MethodSpec) -> list[tuple[int, int, int]]:
    """Contractions the device executes (SYRKs counted as their dense shape).

    UNSO matches the reference (2 long-side products); the quintic step runs
    in the regrouped form X' = aX + (bG + cG^2) X: 2 long-side + 1 short-side."""
    if spec.kind is MethodKind.UNSO:
        return model_matmul_shapes(h, w, spec)
    if spec.kind is MethodKind.ORIGINAL_NS:
        return [(h, w, h), (h, h, w)] * spec.iterations
    return [(h, w, h), (h, h, h), (h, h, w)] * len(spec.quintic_rows())


def expand_cesista_rows(triples) -> np.ndarray:
    """(gamma, r, l) -> (a, b, c) of y + gamma y (y^2-(1+r)^2)(y^2-(1-l)^2) (ortho.py:240-247)."""
    t = np.asarray(triples, dtype=np.float64)
    p = (1.0 + t[:, 1]) ** 2
    q = (1.0 - t[:, 2]) ** 2
    g = t[:, 0]
    return np.column_stack([1.0 + g * p * q, -g * (p + q), g])


def scalar_map(spec: MethodSpec):
    """Composed scalar map applied to each singular value (ortho.py:286-310)."""
    if spec.kind is MethodKind.UNSO:
        coeffs = spec.coeffs
        return lambda x: eval_f(coeffs, x)
    if spec.kind is MethodKind.ORIGINAL_NS:
        its = spec.iterations

        def cubic(x):
            y = np.asarray(x, dtype=np.float64) * 1.0 if not np.isscalar(x) else x
            for _ in range(its):
                y = 0.5 * y * (3.0 - y * y)
            return y
        return cubic
    rows = spec.quintic_rows()

    def quintic(x):
        y = np.asarray(x, dtype=np.float64) * 1.0 if not np.isscalar(x) else x
        for a, b, c in rows:
            yy = y * y
            y = y * (a + b * yy + c * yy * yy)
        return y
    return quintic


# ---------------------------------------------------------------------------- descriptors

_DTYPES = {torch.float32: N.DTYPE_F32, torch.bfloat16: N.DTYPE_BF16, torch.float64: N.DTYPE_F64}
_SCALING = {Scaling.FROBENIUS_GRAM: N.SCALING_GRAM, Scaling.FROBENIUS_PLAIN: N.SCALING_PLAIN,
            Scaling.GELFAND: N.SCALING_GELFAND}


def _row_major(t: torch.Tensor) -> torch.Tensor:
    """The kernels read row-major matrices with any row stride (ld) and batch stride; other layouts
    (transposed or column-strided views) are copied, like the reference's np.ascontiguousarray."""
    if isinstance(t, torch.Tensor) and t.dim() in (2, 3) and t.numel() > 0:
        rows, cols = t.shape[-2], t.shape[-1]
        if t.stride(-1) != 1 or (rows > 1 and t.stride(-2) < cols):
            return t.contiguous()
    return t


def _matrix_desc(t: torch.Tensor) -> N.MatrixDesc:
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor on a CUDA device")
    if not t.is_cuda:
        raise ValueError("input must be a CUDA tensor (there is no CPU path)")
    if t.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {t.dtype}; use float32, bfloat16 or float64")
    if t.dim() == 2:
        rows, cols = t.shape
        batch, bstride = 1, rows * (t.stride(0) if rows > 1 else cols)
    elif t.dim() == 3:
        batch, rows, cols = t.shape
        bstride = t.stride(0)
    else:
        raise ShapeError(f"expected a 2-D matrix or a 3-D batch, got ndim={t.dim()}")
    if rows < 1 or cols < 1 or batch < 1:
        raise ShapeError(f"matrix dimensions must be positive, got {tuple(t.shape)}")
    if t.stride(-1) != 1 or (rows > 1 and t.stride(-2) < cols):
        raise ShapeError("rows must be contiguous (stride(-1) == 1); call .contiguous()")
    ld = t.stride(-2) if rows > 1 else cols
    return N.MatrixDesc(rows, cols, ld, batch, bstride, _DTYPES[t.dtype], 0)


def _resolve_precision(spec: MethodSpec, t: torch.Tensor, precision) -> Precision:
    p = precision if precision is not None else spec.precision
    if p is None:
        p = Precision.BF16 if t.dtype == torch.bfloat16 else Precision.FP32
    return Precision(p)


def _method_desc(spec: MethodSpec, precision: Precision, scaling_code: int):
    """(MethodDesc, coefficient array) for the ABI, memoised on the (immutable) spec; the array is
    kept alive with the descriptor that points into it."""
    key = ("desc", precision, scaling_code)
    hit = spec._cache.get(key)
    if hit is None:
        hit = spec._cache[key] = _build_method_desc(spec, precision, scaling_code)
    return hit


def _build_method_desc(spec: MethodSpec, precision: Precision, scaling_code: int):
    if spec.kind is MethodKind.UNSO:
        co = spec.coeffs.device_coefficients()
        method, order, steps = N.METHOD_UNSO, spec.coeffs.order, 0
    elif spec.kind is MethodKind.ORIGINAL_NS:
        co = np.zeros(1)
        method, order, steps = N.METHOD_ORIGINAL_NS, 0, spec.iterations
    else:
        rows = spec.quintic_rows()
        co = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1)
        method, order, steps = N.METHOD_QUINTIC, 0, rows.shape[0]
    co = np.ascontiguousarray(co, dtype=np.float64)
    flags = {None: 0, 1: N.FLAG_SINGLE_TERM_APPLY, 2: N.FLAG_TWO_TERM_APPLY}[spec.apply_terms]
    if spec.ns_products == "bf16":
        flags |= N.FLAG_NS_SINGLE_STATE
    if spec.chain == "bf16x3":
        flags |= N.FLAG_CHAIN_BF16X3
    if not spec.truncate:
        flags |= N.FLAG_NO_TRUNCATION
    if spec.fp32_engine == "dmma":
        flags |= N.FLAG_FP32_DMMA
    md = N.MethodDesc(method, scaling_code, spec.gelfand_power,
                      N.PREC_BF16 if precision is Precision.BF16 else N.PREC_FP32, order, steps,
                      co.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), flags, 0)
    return md, co  # keep `co` alive for the duration of the call


class _Workspace:
    """Per (device, stream) growable scratch from torch's caching allocator."""

    def __init__(self):
        self._bufs: dict = {}

    def get(self, nbytes: int, device: torch.device, stream: torch.cuda.Stream) -> torch.Tensor:
        key = (device.index, stream.cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf

    def clear(self) -> None:
        self._bufs.clear()


workspace_pool = _Workspace()


def _status_check(status: torch.Tensor | None, check: bool) -> None:
    if check and status is not None and bool((status != 0).any().item()):
        bad = torch.nonzero(status).flatten().tolist()
        raise DegenerateInputError(
            f"matrices {bad}: input is identically zero or the scaling denominator is not a positive finite number")


def _run(m: torch.Tensor, spec: MethodSpec, scaling_code: int, precision, out, check: bool):
    m = _row_major(m)
    xd = _matrix_desc(m)
    prec = _resolve_precision(spec, m, precision)
    md, co = _method_desc(spec, prec, scaling_code)
    lib = N.lib()
    nbytes = lib.unso_workspace_size(ctypes.byref(xd), ctypes.byref(md))
    if nbytes == 0:
        N.check(N.ERR_VALUE, "unso_workspace_size")
    device = m.device
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device)
        ws = workspace_pool.get(nbytes, device, stream)
        y = out if out is not None else torch.empty(m.shape, dtype=m.dtype, device=device)
        if y.shape != m.shape or y.dtype != m.dtype or not y.is_contiguous():
            raise ShapeError("out must be a contiguous tensor with the input's shape and dtype")
        # the status words are only read back when checking (the ABI accepts a null status)
        status = torch.zeros(xd.batch, dtype=torch.int32, device=device) if check else None
        code = lib.unso_orthogonalize(ctypes.byref(xd), ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                      ctypes.byref(md), ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                                      ctypes.c_void_p(status.data_ptr() if status is not None else None),
                                      ctypes.c_void_p(stream.cuda_stream))
        launches = N.launch_count()
        info = None
        if code == N.OK and check:
            sc = torch.empty(xd.batch, N.SCALARS, dtype=torch.float64, device=device)
            if lib.unso_query_scalars(ctypes.byref(xd), ctypes.byref(md), ctypes.c_void_p(ws.data_ptr()),
                                      ctypes.c_void_p(sc.data_ptr()), ctypes.c_void_p(stream.cuda_stream)) == N.OK:
                rows = sc.cpu().numpy()
                info = [dict(zip(N.SCALAR_NAMES, map(float, r))) for r in rows]
    del co
    N.check(code, "unso_orthogonalize")
    _status_check(status, check)
    return y, prec, launches, info


def _hw(m: torch.Tensor) -> tuple[int, int, bool]:
    rows, cols = m.shape[-2], m.shape[-1]
    tall = rows > cols
    return (cols, rows, tall) if tall else (rows, cols, tall)


# ---------------------------------------------------------------------------- public API

def orthogonalize(m: torch.Tensor, spec: MethodSpec, *, precision=None, out=None, check: bool = True) -> OrthoResult:
    """preprocess -> kernel -> restore orientation (ortho.py:267-283), fused on the device."""
    h, w, tall = _hw(m)
    scaling = spec.effective_scaling
    y, prec, launches, info = _run(m, spec, _SCALING[scaling], precision, out, check)
    key = ("model", h, w)
    meta = spec._cache.get(key)
    if meta is None:
        meta = spec._cache[key] = (kernel_model_flops(h, w, spec),
                                   preprocess_model_flops(h, w, scaling, spec.gelfand_power),
                                   model_matmul_shapes(h, w, spec), executed_matmul_shapes(h, w, spec))
    return OrthoResult(y=y, flops=meta[0], was_transposed=tall, preprocess_flops=meta[1],
                       kernel_matmul_shapes=list(meta[2]), executed_matmul_shapes=list(meta[3]),
                       precision=prec.value, launches=launches, info=info)


def scale_denominator(m: torch.Tensor, scaling: Scaling, gelfand_power: int = 2, check: bool = True) -> torch.Tensor:
    """Per-matrix preprocess denominator on the device (ortho.py:153-165), float64 tensor."""
    m = _row_major(m)
    xd = _matrix_desc(m)
    scaling = Scaling(scaling)
    md = N.MethodDesc(N.METHOD_UNSO, _SCALING[scaling], gelfand_power, N.PREC_FP32, 1, 0, None, 0, 0)
    lib = N.lib()
    dummy = N.MethodDesc(N.METHOD_UNSO, _SCALING[scaling], gelfand_power, N.PREC_FP32, 1, 0,
                         (ctypes.c_double * 1)(0.0), 0, 0)
    nbytes = lib.unso_workspace_size(ctypes.byref(xd), ctypes.byref(dummy))
    with torch.cuda.device(m.device):
        stream = torch.cuda.current_stream(m.device)
        ws = workspace_pool.get(nbytes, m.device, stream)
        denom = torch.empty(xd.batch, dtype=torch.float64, device=m.device)
        status = torch.zeros(xd.batch, dtype=torch.int32, device=m.device)
        code = lib.unso_scale_denominator(ctypes.byref(xd), ctypes.c_void_p(m.data_ptr()), ctypes.byref(md),
                                          ctypes.c_void_p(denom.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                          ctypes.c_size_t(ws.numel()), ctypes.c_void_p(status.data_ptr()),
                                          ctypes.c_void_p(stream.cuda_stream))
    N.check(code, "unso_scale_denominator")
    _status_check(status, check)
    return denom


def preprocess(m: torch.Tensor, scaling: Scaling, counter: FlopsCounter | None = None,
               gelfand_power: int = 2) -> tuple[torch.Tensor, bool]:
    """Orient row-wide and rescale so every singular value is in [0, 1] (ortho.py:140-168).

    Returns a new tensor (a transposed copy when tall), like the reference."""
    h, w, tall = _hw(m)
    denom = scale_denominator(m, scaling, gelfand_power)
    if counter is not None:
        counter.add(preprocess_model_flops(h, w, scaling, gelfand_power) - (2 * h * h * w if
                    Scaling(scaling) is not Scaling.FROBENIUS_PLAIN else 0))
        if Scaling(scaling) is not Scaling.FROBENIUS_PLAIN:
            counter.record_matmul(h, w, h)
    a = m.transpose(-1, -2) if tall else m
    shape = (-1, 1, 1) if m.dim() == 3 else ()
    # The reference keeps the rescaled copy in fp64 (ortho.py:167).  A bf16 input is returned as
    # fp32 (exact: bf16 x fp64 scale rounded once to fp32, 24 significant bits) so that
    # unso(preprocess(x)) computes on the same values as the fused orthogonalize path instead of a
    # twice-rounded bf16 copy; fp32 / fp64 inputs keep their dtype.
    out_dtype = torch.float32 if m.dtype == torch.bfloat16 else m.dtype
    x = (a.to(torch.float64) / denom.view(shape)).to(out_dtype).contiguous()
    return x, tall


def _bare(x: torch.Tensor, spec: MethodSpec, counter, precision, check=False) -> torch.Tensor:
    h, w = x.shape[-2], x.shape[-1]
    if h > w:
        raise ShapeError(f"kernel expects rows <= cols, got {h}x{w}")  # ortho.py:186-187, 211-212, 223-224
    y, _, _, _ = _run(x, spec, N.SCALING_NONE, precision, None, check)
    if counter is not None:
        for s in model_matmul_shapes(h, w, spec):
            counter.matmul_shapes.append(s)
        counter.add(kernel_model_flops(h, w, spec))
    return y


def unso(x: torch.Tensor, coeffs: CoefficientSet, counter: FlopsCounter | None = None, debug: bool = False,
         *, precision=None) -> torch.Tensor:
    """Single-pass polynomial on a row-wide, pre-scaled input (ortho.py:171-205)."""
    if debug:
        top = float(torch.linalg.matrix_norm(x.double(), ord=2).max())
        if top > 1.0 + 1e-9:
            warnings.warn(f"input has a singular value {top:.6g} above 1; result may be inaccurate",
                          RuntimeWarning, stacklevel=2)
    return _bare(x, MethodSpec(MethodKind.UNSO, coeffs=coeffs), counter, precision)


def original_ns(x: torch.Tensor, iterations: int, counter: FlopsCounter | None = None, *,
                precision=None) -> torch.Tensor:
    """X <- 0.5 (3I - X X^T) X, iterated (ortho.py:208-218)."""
    return _bare(x, MethodSpec(MethodKind.ORIGINAL_NS, iterations=iterations), counter, precision)


def muon_ns(x: torch.Tensor, iterations: int, counter: FlopsCounter | None = None, *,
            precision=None) -> torch.Tensor:
    """Fixed-coefficient quintic iteration (ortho.py:234-237)."""
    return _bare(x, MethodSpec(MethodKind.MUON_NS, iterations=iterations), counter, precision)


def cesista_ns(x: torch.Tensor, step_params: CesistaStepParams, counter: FlopsCounter | None = None, *,
               precision=None) -> torch.Tensor:
    """Per-step reparameterised quintic iteration (ortho.py:250-256)."""
    return _bare(x, MethodSpec(MethodKind.CESISTA_NS, step_params=step_params), counter, precision)


def ortho_error_device(y: torch.Tensor) -> torch.Tensor:
    """||Y Y^T - I||_F on the short side, per matrix, as a float64 CUDA tensor (bench.py:71-82)."""
    y = _row_major(y)
    yd = _matrix_desc(y)
    lib = N.lib()
    md = N.MethodDesc(N.METHOD_UNSO, N.SCALING_GRAM, 1, N.PREC_FP32, 1, 0, (ctypes.c_double * 1)(0.0), 0, 0)
    nbytes = lib.unso_workspace_size(ctypes.byref(yd), ctypes.byref(md))
    with torch.cuda.device(y.device):
        stream = torch.cuda.current_stream(y.device)
        ws = workspace_pool.get(nbytes, y.device, stream)
        err = torch.empty(yd.batch, dtype=torch.float64, device=y.device)
        code = lib.unso_ortho_error(ctypes.byref(yd), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(err.data_ptr()),
                                    ctypes.c_void_p(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                                    ctypes.c_void_p(stream.cuda_stream))
    N.check(code, "unso_ortho_error")
    return err


def ortho_error(y: torch.Tensor) -> float:
    """bench.py:71-77 (row-wide input required, like the reference)."""
    if y.shape[-2] > y.shape[-1]:
        raise ShapeError(f"ortho_error expects rows <= cols, got {y.shape[-2]}x{y.shape[-1]}")
    e = ortho_error_device(y)
    return float(e[0]) if e.numel() == 1 else e.cpu().tolist()


def ortho_error_any(y: torch.Tensor):
    """bench.py:80-82: short-side orientation chosen automatically."""
    e = ortho_error_device(y)
    return float(e[0]) if e.numel() == 1 else e.cpu().tolist()
