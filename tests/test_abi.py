"""The C-ABI library loads and exports every symbol include/unso_b200.h declares;
host-side validation paths return the documented status codes.  No GPU needed
(no compute call is made)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2602_02500_b200 import _native as N

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(REPO, "include", "unso_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(unso_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    assert sorted(N.EXPORTED_SYMBOLS) == syms
    for s in syms:
        assert hasattr(lib, s), s
    assert "sm_100a" in N.version()


def test_library_is_sm100a_cubin():
    """The fat binary carries sm_100a SASS with tcgen05 MMAs and TMA loads."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", N.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out      # tcgen05.mma kind::f16
    assert "UTCIMMA" in out      # tcgen05.mma kind::i8 (fp32 mode digit products)
    assert "UTMALDG.4D" in out   # 4-D TMA box of the int8 digit planes
    assert "UTMALDG" in out      # TMA tensor loads
    assert "LDTM" in out         # tcgen05.ld


def _desc(rows, cols, ld=None, batch=1, dtype=N.DTYPE_F32):
    return N.MatrixDesc(rows, cols, ld or cols, batch, rows * (ld or cols), dtype, 0)


def _method(method=N.METHOD_UNSO, order=14, steps=0, prec=N.PREC_FP32, scaling=N.SCALING_GRAM):
    co = (ctypes.c_double * max(order, 3 * max(steps, 1)))(*([0.5] * max(order, 3 * max(steps, 1))))
    return N.MethodDesc(method, scaling, 2, prec, order, steps, ctypes.cast(co, ctypes.POINTER(ctypes.c_double)), 0, 0), co


def test_workspace_size_and_validation():
    lib = N.lib()
    md, co = _method()
    x = _desc(512, 128)
    assert lib.unso_workspace_size(ctypes.byref(x), ctypes.byref(md)) > 0
    bad = _desc(0, 128)
    assert lib.unso_workspace_size(ctypes.byref(bad), ctypes.byref(md)) == 0
    # invalid shape / values are rejected on the host, before any CUDA call
    code = lib.unso_orthogonalize(ctypes.byref(bad), None, None, ctypes.byref(md), None, 0, None, None)
    assert code == N.ERR_SHAPE
    md2, co2 = _method(order=0)
    code = lib.unso_orthogonalize(ctypes.byref(x), ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.byref(md2),
                                  None, 0, None, None)
    assert code == N.ERR_VALUE
    code = lib.unso_orthogonalize(ctypes.byref(x), ctypes.c_void_p(256), ctypes.c_void_p(256), ctypes.byref(md),
                                  None, 0, None, None)
    assert code == N.ERR_WORKSPACE
    # NS methods in BF16 precision are not implemented in this build
    md3, co3 = _method(method=N.METHOD_QUINTIC, order=0, steps=5, prec=N.PREC_BF16, scaling=N.SCALING_PLAIN)
    code = lib.unso_orthogonalize(ctypes.byref(x), ctypes.c_void_p(256), ctypes.c_void_p(256), ctypes.byref(md3),
                                  None, 0, None, None)
    assert code in (N.ERR_UNSUPPORTED, N.OK, N.ERR_WORKSPACE)


def test_status_strings_and_exception_mapping():
    assert N.status_message(N.OK) == "ok"
    from paper_2602_02500_b200.errors import DegenerateInputError, ShapeError
    with pytest.raises(ShapeError):
        N.check(N.ERR_SHAPE, "x")
    with pytest.raises(DegenerateInputError):
        N.check(N.ERR_DEGENERATE, "x")
    assert N.lib().unso_gram_dtype(None) == N.DTYPE_F64


def test_no_oracle_import_in_product():
    """The product package never imports the oracle (no CPU fallback)."""
    pkg = os.path.join(REPO, "paper_2602_02500_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_gram_peer_buffer_sizes():
    """unso_gram_peer_bytes (host-only): slot buffer = world x splits x ceil(tiles / world) 256x256 fp32
    tiles, Gram = h^2 fp32, flags = 2 x world words; invalid arguments give 0."""
    lib = N.lib()
    for h, world, splits in ((2048, 8, 2), (512, 4, 4), (640, 3, 1), (128, 1, 1)):
        nt = (h + 255) // 256
        tiles = nt * (nt + 1) // 2
        owned = -(-tiles // world)
        assert lib.unso_gram_peer_bytes(h, world, splits, 0) == world * splits * owned * 256 * 256 * 4
        assert lib.unso_gram_peer_bytes(h, world, splits, 1) == h * h * 4
        assert lib.unso_gram_peer_bytes(h, world, splits, 2) == 2 * world * 4
    assert lib.unso_gram_peer_bytes(2048, 9, 1, 0) == 0
    assert lib.unso_gram_peer_bytes(2048, 2, 0, 0) == 0
    from paper_2602_02500_b200.distributed import gram_push_splits
    assert gram_push_splits(2048, 32768) == 2 and gram_push_splits(128, 64) == 1


def test_header_constants_match_the_binding():
    """Every enum value and #define of include/unso_b200.h equals the ctypes binding's constant
    (guards the ABI against drift between the header and _native.py)."""
    import re
    from paper_2602_02500_b200 import _native as N
    text = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                             "unso_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    consts = {m.group(1): int(m.group(2), 0) for m in re.finditer(r"\b(UNSO_[A-Z0-9_]+)\s*=\s*(0x[0-9a-fA-F]+|\d+)", text)}
    consts.update({m.group(1): int(m.group(2), 0)
                   for m in re.finditer(r"#define\s+(UNSO_[A-Z0-9_]+)\s+(0x[0-9a-fA-F]+|\d+)", text)})
    expect = {
        "UNSO_OK": N.OK, "UNSO_ERR_SHAPE": N.ERR_SHAPE, "UNSO_ERR_DEGENERATE": N.ERR_DEGENERATE,
        "UNSO_ERR_VALUE": N.ERR_VALUE, "UNSO_ERR_CUDA": N.ERR_CUDA, "UNSO_ERR_UNSUPPORTED": N.ERR_UNSUPPORTED,
        "UNSO_ERR_WORKSPACE": N.ERR_WORKSPACE,
        "UNSO_DTYPE_F32": N.DTYPE_F32, "UNSO_DTYPE_BF16": N.DTYPE_BF16, "UNSO_DTYPE_F64": N.DTYPE_F64,
        "UNSO_PREC_FP32": N.PREC_FP32, "UNSO_PREC_BF16": N.PREC_BF16,
        "UNSO_SCALING_GRAM": N.SCALING_GRAM, "UNSO_SCALING_PLAIN": N.SCALING_PLAIN,
        "UNSO_SCALING_GELFAND": N.SCALING_GELFAND, "UNSO_SCALING_NONE": N.SCALING_NONE,
        "UNSO_METHOD_UNSO": N.METHOD_UNSO, "UNSO_METHOD_ORIGINAL_NS": N.METHOD_ORIGINAL_NS,
        "UNSO_METHOD_QUINTIC": N.METHOD_QUINTIC,
        "UNSO_FLAG_SINGLE_TERM_APPLY": N.FLAG_SINGLE_TERM_APPLY, "UNSO_FLAG_TWO_TERM_APPLY": N.FLAG_TWO_TERM_APPLY,
        "UNSO_FLAG_CHAIN_BF16X3": N.FLAG_CHAIN_BF16X3, "UNSO_FLAG_NO_TRUNCATION": N.FLAG_NO_TRUNCATION,
        "UNSO_FLAG_NS_SINGLE_STATE": N.FLAG_NS_SINGLE_STATE, "UNSO_FLAG_FP32_DMMA": N.FLAG_FP32_DMMA,
        "UNSO_MAX_PEERS": N.MAX_PEERS, "UNSO_SCALARS": N.SCALARS, "UNSO_PROFILE_STAGES": len(N.PROFILE_STAGES),
    }
    for name, value in expect.items():
        assert consts.get(name) == value, (name, consts.get(name), value)
