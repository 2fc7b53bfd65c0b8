"""C-ABI boundary checks that need no GPU: the library loads, exports every entry point that
include/jigsaw_sm100.h declares, reports its version, and rejects bad shapes with the
reference's exception types before touching the device."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "jigsaw_sm100.h")
LIB = os.path.join(ROOT, "paper_2507_05753_b200", "libjigsaw_sm100.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|int64_t|size_t)\s+(jg_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2507_05753_b200.csrc.build import build
        build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("jg_gemm", "jg_epilogue", "jg_ln_apply", "jg_ln_bwd_apply", "jg_blend_loss", "jg_adam",
                 "jg_patchify", "jg_unpatchify", "jg_version", "jg_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_table_matches_header():
    from paper_2507_05753_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_version_and_error_strings(lib):
    lib.jg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.jg_version()


def test_shape_errors_raise_before_launch(lib):
    """Shape validation happens on the host: a bad descriptor returns JG_ERR_SHAPE with a message."""
    from paper_2507_05753_b200 import _lib
    from paper_2507_05753_b200.errors import ShapeError
    _lib.load(LIB)
    d = _lib.GemmDesc()
    d.m, d.n, d.k, d.batch = 0, 8, 8, 1  # empty problem
    with pytest.raises(ShapeError, match="empty problem"):
        _lib._check(_lib.load().jg_gemm(ctypes.byref(d), None), "jg_gemm")
    with pytest.raises(ShapeError, match="eps"):
        _lib._check(_lib.load().jg_ln_apply(None, None, None, None, None, 0, None, 4, 4, 4, ctypes.c_float(0.0), None, None),
                    "jg_ln_apply")
    with pytest.raises(ShapeError, match="not divisible"):
        _lib._check(_lib.load().jg_patchify(None, None, 0, 1, 5, 8, 2, 2, 2, None), "jg_patchify")


def test_gemm_desc_layout_matches_binding(lib):
    """The ctypes mirror of jg_gemm_desc has the library's size (a stale .so or a field added on
    one side only is caught at load time by _lib.load, and here without a GPU)."""
    from paper_2507_05753_b200 import _lib
    lib.jg_gemm_desc_size.restype = ctypes.c_size_t
    assert lib.jg_gemm_desc_size() == ctypes.sizeof(_lib.GemmDesc)
