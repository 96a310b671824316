"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re

import numpy as np

from paper_2504_07264_b200 import _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "splitfft_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfft_\w+)\s*\(", text)))


def test_header_declares_the_expected_entry_points():
    syms = declared_symbols()
    for name in ("sfft_plan_create", "sfft_plan_destroy", "sfft_exec_split", "sfft_exec_interleaved",
                 "sfft_workspace_bytes", "sfft_last_error", "sfft_abi_version"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_ffi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"not exported: {missing}"
    assert set(declared_symbols()) == set(_ffi.SIGNATURES), "ctypes table out of sync with the header"


def test_abi_version_and_error_reporting():
    assert _ffi.lib.sfft_abi_version() == _ffi.ABI_VERSION
    wr = np.zeros(4)
    assert _ffi.lib.sfft_twiddle_table(0, wr.ctypes.data, wr.ctypes.data) == _ffi.SFFT_EINVAL
    assert b"log2n" in _ffi.lib.sfft_last_error()


def test_plan_create_validates_before_touching_the_device():
    h = ctypes.c_void_p()
    assert _ffi.lib.sfft_plan_create(-1, 0, 0, 0, 30, ctypes.byref(h)) == _ffi.SFFT_EINVAL
    assert b"must be >= 0" in _ffi.lib.sfft_last_error()
    assert _ffi.lib.sfft_plan_create(12, 0, 0, 0, 10, ctypes.byref(h)) == _ffi.SFFT_ECAPACITY
    assert b"exceeds the plan limit" in _ffi.lib.sfft_last_error()
    assert _ffi.lib.sfft_plan_create(5, 0, 7, 0, 30, ctypes.byref(h)) == _ffi.SFFT_EINVAL
    assert _ffi.lib.sfft_exec_split(None, None, None, None, None, 1, 8, 8, -1, None, None) == _ffi.SFFT_EINVAL


def test_launch_counter_is_exported():
    assert _ffi.launch_count() >= 0


def test_plan_create_validates_the_large_path_kernel_choice():
    # kernel 'pass' (one launch per group) needs log2n > 12, 'pass2' (the
    # L2-fused group pairs) 20 <= log2n <= 28; checked before any device call
    h = ctypes.c_void_p()
    rc = _ffi.lib.sfft_plan_create_ex(12, 0, 0, 0, 30, 0, _ffi.SFFT_KERNEL_PASS, ctypes.byref(h))
    assert rc == _ffi.SFFT_EINVAL and b"log2n > 12" in _ffi.lib.sfft_last_error()
    for m in (19, 29):
        rc = _ffi.lib.sfft_plan_create_ex(m, 0, 0, 0, 30, 0, _ffi.SFFT_KERNEL_PASS2, ctypes.byref(h))
        assert rc == _ffi.SFFT_EINVAL and b"20 <= log2n <= 28" in _ffi.lib.sfft_last_error()
    rc = _ffi.lib.sfft_plan_create_ex(20, 0, 0, 0, 30, 0, 5, ctypes.byref(h))
    assert rc == _ffi.SFFT_EINVAL and b"unknown kernel family" in _ffi.lib.sfft_last_error()
