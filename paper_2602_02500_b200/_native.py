"""ctypes binding of the C ABI in ``include/unso_b200.h`` (``libunso_b200.so``).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or fails to load, every entry point raises ``NativeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DegenerateInputError, NativeError, ShapeError, UnsupportedError

LIB_NAME = "libunso_b200.so"
LIB_PATH = os.environ.get("UNSO_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# unso_status
OK, ERR_SHAPE, ERR_DEGENERATE, ERR_VALUE, ERR_CUDA, ERR_UNSUPPORTED, ERR_WORKSPACE = range(7)
# unso_dtype
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2
# unso_precision
PREC_FP32, PREC_BF16 = 0, 1
# unso_scaling
SCALING_GRAM, SCALING_PLAIN, SCALING_GELFAND, SCALING_NONE = 0, 1, 2, 3
# unso_method
METHOD_UNSO, METHOD_ORIGINAL_NS, METHOD_QUINTIC = 0, 1, 2
FLAG_SINGLE_TERM_APPLY = 0x1

#: every symbol include/unso_b200.h declares
EXPORTED_SYMBOLS = (
    "unso_version", "unso_status_string", "unso_workspace_size", "unso_orthogonalize", "unso_gram",
    "unso_gram_dtype", "unso_orthogonalize_from_gram", "unso_scale_denominator", "unso_ortho_error",
    "unso_last_launch_count", "unso_profile_begin", "unso_profile_read", "unso_profile_end",
    "unso_query_scalars", "unso_gram_peer_bytes", "unso_gram_push", "unso_gram_reduce", "unso_gram_wait",
    "unso_muon_prepare", "unso_muon_update",
)
SCALARS = 16
SCALAR_NAMES = ("trace", "fro2", "dev2", "s2", "inv_s", "ortho_error", "shift", "apply_single", "apply_bound",
                "chain_steps")
FLAG_TWO_TERM_APPLY = 0x2
FLAG_NO_TRUNCATION = 0x8
FLAG_CHAIN_BF16X3 = 0x4
FLAG_NS_SINGLE_STATE = 0x10
FLAG_FP32_DMMA = 0x20
PROFILE_STAGES = ("convert", "gram", "scale_prep", "chain", "finalize_p", "apply")


class MatrixDesc(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("batch", ctypes.c_int64), ("batch_stride", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("orientation", ctypes.c_int32)]


class MethodDesc(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("scaling", ctypes.c_int32), ("gelfand_power", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("order", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("coeffs", ctypes.POINTER(ctypes.c_double)), ("flags", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


MAX_PEERS = 8


class GramPeers(ctypes.Structure):
    """unso_gram_peers: every rank's peer-mapped slot / Gram / flag buffers."""
    _fields_ = [("slots", ctypes.c_void_p * MAX_PEERS), ("g", ctypes.c_void_p * MAX_PEERS),
                ("flags", ctypes.c_void_p * MAX_PEERS)]


_lib = None
_lock = threading.Lock()


def _declare(lib: ctypes.CDLL) -> None:
    P = ctypes.c_void_p
    MD, XD = ctypes.POINTER(MethodDesc), ctypes.POINTER(MatrixDesc)
    lib.unso_version.restype = ctypes.c_char_p
    lib.unso_version.argtypes = []
    lib.unso_status_string.restype = ctypes.c_char_p
    lib.unso_status_string.argtypes = [ctypes.c_int32]
    lib.unso_workspace_size.restype = ctypes.c_size_t
    lib.unso_workspace_size.argtypes = [XD, MD]
    lib.unso_orthogonalize.restype = ctypes.c_int32
    lib.unso_orthogonalize.argtypes = [XD, P, P, MD, P, ctypes.c_size_t, P, P]
    lib.unso_gram.restype = ctypes.c_int32
    lib.unso_gram.argtypes = [XD, P, P, MD, P, ctypes.c_size_t, P]
    lib.unso_gram_dtype.restype = ctypes.c_int32
    lib.unso_gram_dtype.argtypes = [MD]
    lib.unso_orthogonalize_from_gram.restype = ctypes.c_int32
    lib.unso_orthogonalize_from_gram.argtypes = [XD, P, P, P, MD, P, ctypes.c_size_t, P, P]
    lib.unso_scale_denominator.restype = ctypes.c_int32
    lib.unso_scale_denominator.argtypes = [XD, P, MD, P, P, ctypes.c_size_t, P, P]
    lib.unso_ortho_error.restype = ctypes.c_int32
    lib.unso_ortho_error.argtypes = [XD, P, P, P, ctypes.c_size_t, P]
    lib.unso_last_launch_count.restype = ctypes.c_int32
    lib.unso_last_launch_count.argtypes = []
    lib.unso_profile_begin.restype = ctypes.c_int32
    lib.unso_profile_begin.argtypes = [ctypes.c_int32]
    lib.unso_profile_read.restype = ctypes.c_int32
    lib.unso_profile_read.argtypes = [P, ctypes.c_int32]
    lib.unso_query_scalars.restype = ctypes.c_int32
    lib.unso_query_scalars.argtypes = [XD, MD, P, P, P]
    lib.unso_profile_end.restype = None
    lib.unso_profile_end.argtypes = []
    GP = ctypes.POINTER(GramPeers)
    lib.unso_gram_peer_bytes.restype = ctypes.c_size_t
    lib.unso_gram_peer_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
    lib.unso_gram_push.restype = ctypes.c_int32
    lib.unso_gram_push.argtypes = [XD, P, MD, GP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                                   P, ctypes.c_size_t, P]
    lib.unso_gram_reduce.restype = ctypes.c_int32
    lib.unso_gram_reduce.argtypes = [ctypes.c_int64, GP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_uint32, P, ctypes.c_size_t, P]
    lib.unso_muon_prepare.restype = ctypes.c_int32
    lib.unso_muon_prepare.argtypes = [ctypes.c_int32, P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_float,
                                      ctypes.c_int32, P, P]
    lib.unso_muon_update.restype = ctypes.c_int32
    lib.unso_muon_update.argtypes = [ctypes.c_int32, P, P, ctypes.c_int64, ctypes.c_int32, P, ctypes.c_float,
                                     ctypes.c_float, P]
    lib.unso_gram_wait.restype = ctypes.c_int32
    lib.unso_gram_wait.argtypes = [ctypes.c_int64, GP, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, P]


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raise NativeError if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            try:
                handle = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(handle)
            _lib = handle
    return _lib


def status_message(code: int) -> str:
    return lib().unso_status_string(int(code)).decode()


def check(code: int, what: str) -> None:
    """Map an unso_status onto the reference's exception types."""
    if code == OK:
        return
    msg = f"{what}: {status_message(code)}"
    if code == ERR_SHAPE:
        raise ShapeError(msg)
    if code == ERR_DEGENERATE:
        raise DegenerateInputError(msg)
    if code == ERR_VALUE:
        raise ValueError(msg)
    if code == ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise NativeError(msg)


def version() -> str:
    return lib().unso_version().decode()


def launch_count() -> int:
    return int(lib().unso_last_launch_count())


class StageProfiler:
    """Context manager around unso_profile_*: per-call stage times (ms) of
    unso_orthogonalize, recorded with CUDA events on the call's stream."""

    def __init__(self, max_calls: int):
        self.max_calls = max_calls
        self.times = None

    def __enter__(self):
        check(lib().unso_profile_begin(self.max_calls), "unso_profile_begin")
        return self

    def read(self):
        import numpy as np
        buf = (ctypes.c_float * (self.max_calls * len(PROFILE_STAGES)))()
        n = lib().unso_profile_read(ctypes.cast(buf, ctypes.c_void_p), self.max_calls)
        arr = np.frombuffer(buf, dtype=np.float32).reshape(self.max_calls, len(PROFILE_STAGES))[:n].copy()
        self.times = arr
        return arr

    def __exit__(self, *exc):
        if self.times is None:
            self.read()
        lib().unso_profile_end()
        return False
