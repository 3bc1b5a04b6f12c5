"""B200-native UNSO orthogonalization (arXiv 2602.02500 hot path).

Drop-in for the reference package's orthogonalization entry points
(``unso.ortho`` / ``unso.scalarpoly``, re-exported like unso/__init__.py:4-100),
operating on CUDA tensors.  All matrix arithmetic runs in the in-tree CUDA
library ``libunso_b200.so`` (sm_100a: tcgen05/TMEM/TMA + fp64 DMMA parity path);
there is no CPU fallback.
"""

from .errors import DegenerateInputError, NativeError, ParseError, ShapeError, UnsupportedError
from .ortho import (
    DEFAULT_MUON_ITERATIONS,
    DEFAULT_ORIGINAL_ITERATIONS,
    MUON_COEFFICIENTS,
    FlopsCounter,
    MethodKind,
    MethodSpec,
    OrthoResult,
    Precision,
    Scaling,
    cesista_ns,
    executed_matmul_shapes,
    expand_cesista_rows,
    kernel_model_flops,
    model_matmul_shapes,
    muon_ns,
    original_ns,
    ortho_error,
    ortho_error_any,
    ortho_error_device,
    orthogonalize,
    preprocess,
    preprocess_model_flops,
    scalar_map,
    scale_denominator,
    unso,
)
from .muon import Muon
from .scalarpoly import (
    BRule,
    CesistaStepParams,
    CoefficientSet,
    constraint_point,
    constraint_residual,
    default_cesista_triples,
    default_coefficients,
    derive_b,
    eval_f,
    read_coefficients,
    read_step_triples,
    write_coefficients,
)

__all__ = [
    "Muon", "BRule", "CesistaStepParams", "CoefficientSet", "DEFAULT_MUON_ITERATIONS", "DEFAULT_ORIGINAL_ITERATIONS",
    "DegenerateInputError", "FlopsCounter", "MUON_COEFFICIENTS", "MethodKind", "MethodSpec", "NativeError",
    "OrthoResult", "ParseError", "Precision", "Scaling", "ShapeError", "UnsupportedError", "cesista_ns",
    "constraint_point", "constraint_residual", "default_cesista_triples", "default_coefficients", "derive_b",
    "eval_f", "executed_matmul_shapes", "expand_cesista_rows", "kernel_model_flops", "model_matmul_shapes",
    "muon_ns", "original_ns", "ortho_error", "ortho_error_any", "ortho_error_device", "orthogonalize",
    "preprocess", "preprocess_model_flops", "read_coefficients", "read_step_triples", "scalar_map",
    "scale_denominator", "unso", "write_coefficients",
]

__version__ = "0.1.0"
