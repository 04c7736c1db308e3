"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/qadapter.h
declares, reports its version, and rejects bad arguments before touching the device."""

import ctypes
import os
import re

import pytest

from paper_2402_13533_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "qadapter.h")).read()
    return sorted(set(re.findall(r"QA_API\s+[\w\s\*]+?\b(qa_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    syms = _header_symbols()
    assert len(syms) >= 10
    assert sorted(_lib.EXPORTS) == syms


def test_library_exports_every_symbol():
    lib = _lib.lib()
    for s in _header_symbols():
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.qa_version()


def test_argument_validation_without_device():
    lib = _lib.lib()
    # bits outside {4, 8} -> QA_ERR_BITS before any CUDA call (quant.py:74-75)
    st = lib.qa_quantize_rows(None, 0, 1, 1, 1, 3, None, 1, 1, None, None, None, None, None)
    assert st == _lib.QA_ERR_BITS
    assert b"bits" in lib.qa_last_error()
    st = lib.qa_quantize_rows(None, 0, 1, 1, 1, 8, None, 1, 1, None, None, None, None, None)
    assert st == _lib.QA_ERR_ARG
    w = _lib.QWeight(0, 0, 8, None, None, None, None)
    assert lib.qa_linear_workspace_bytes(ctypes.byref(w), None, 16) == 0


def test_workspace_query_and_tt_validation():
    lib = _lib.lib()
    dummy = 16
    w = _lib.QWeight(4096, 4096, 8, dummy, dummy, dummy, dummy)
    base = lib.qa_linear_workspace_bytes(ctypes.byref(w), None, 16384)
    assert base >= 16384 * 4096  # act codes at least
    tt = _lib.TT()
    tt.d = 3
    for k, (m, n) in enumerate(((1, 256), (16, 4), (256, 4))):
        tt.m[k], tt.n[k], tt.cores[k] = m, n, dummy
    for k, r in enumerate((1, 8, 8, 1)):
        tt.r[k] = r
    with_tt = lib.qa_linear_workspace_bytes(ctypes.byref(w), ctypes.byref(tt), 16384)
    assert with_tt > base
    tt.m[2] = 128  # modes no longer multiply to the base shape -> rejected
    assert lib.qa_linear_workspace_bytes(ctypes.byref(w), ctypes.byref(tt), 16384) == 0
    assert b"TT modes" in lib.qa_last_error()
