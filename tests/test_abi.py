"""The drop-in boundary on CPU: libgpp_b200.so loads without a GPU and exports every
entry point include/gpp_b200.h declares, and the ctypes binding (runtime/lib.py) types
exactly those symbols.  No compute calls (there is no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpp_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)  # drop comments (they name symbols too)
    return sorted(set(re.findall(r"\b(gpp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so():
    from paper_2406_17145_b200 import _build

    path = _build.build()
    return ctypes.CDLL(str(path))


def test_library_exports_every_declared_symbol(so):
    names = _declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_ctypes_binding_covers_the_header():
    from paper_2406_17145_b200.runtime import lib

    assert sorted(lib._SIGS) == _declared()


def test_last_error_is_callable_without_gpu(so):
    so.gpp_last_error.restype = ctypes.c_char_p
    assert isinstance(so.gpp_last_error(), bytes)


def test_argument_errors_are_reported_not_crashed(so):
    """A bad shape returns GPP_ERR_ARG (1) with a message, before any CUDA call."""
    so.gpp_last_error.restype = ctypes.c_char_p
    f = so.gpp_attn_fwd
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 5 + [ctypes.c_float, ctypes.c_void_p]
    f.restype = ctypes.c_int
    buf = ctypes.create_string_buffer(64)
    p = ctypes.cast(buf, ctypes.c_void_p)
    assert f(p, p, p, 64, 1, 100, 64, 1, 0.125, None) == 1  # S = 100 unsupported
    assert b"S in" in so.gpp_last_error()
