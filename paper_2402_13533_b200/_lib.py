"""ctypes binding of libqadapter.so (include/qadapter.h).

The library is the product: there is no Python / CPU fallback.  Loading fails loudly
when the shared object is missing or was built for another ABI.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QADAPTER_LIB", os.path.join(HERE, "libqadapter.so"))

QA_OK = 0
QA_ERR_ARG = -1
QA_ERR_BITS = -2
QA_ERR_CUDA = -3
QA_ERR_UNSUPPORTED = -4
QA_ERR_WORKSPACE = -5
QA_F32 = 0
QA_BF16 = 1
QA_TT_MAX_D = 4

EXPORTS = (
    "qa_version",
    "qa_last_error",
    "qa_quantize_rows",
    "qa_dequantize_rows",
    "qa_code_rowsum",
    "qa_qmatmul_workspace_bytes",
    "qa_qmatmul",
    "qa_qmatmul_t",
    "qa_rmsnorm_forward",
    "qa_rmsnorm_backward",
    "qa_rope",
    "qa_swiglu_forward",
    "qa_swiglu_backward",
    "qa_cross_entropy",
    "qa_mse",
    "qa_linear_workspace_bytes",
    "qa_linear_forward",
    "qa_linear_backward",
    "qa_linear_saved_bytes",
    "qa_linear_forward_save",
    "qa_linear_backward_saved",
    "qa_group_workspace_bytes",
    "qa_group_forward",
    "qa_group_backward",
    "qa_adamw_step",
    "qa_nonfinite_segments",
    "qa_merge_workspace_bytes",
    "qa_merge",
    "qa_tt_materialize",
    "qa_gemm_bf16",
    "qa_launch_count",
    "qa_timing_enable",
    "qa_timing_read",
)


class QWeight(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("bits", ctypes.c_int32),
        ("codes", ctypes.c_void_p),
        ("scale", ctypes.c_void_p),
        ("offset", ctypes.c_void_p),
        ("rowsum", ctypes.c_void_p),
    ]


class TT(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32),
        ("m", ctypes.c_int32 * QA_TT_MAX_D),
        ("n", ctypes.c_int32 * QA_TT_MAX_D),
        ("r", ctypes.c_int32 * (QA_TT_MAX_D + 1)),
        ("cores", ctypes.c_void_p * QA_TT_MAX_D),
    ]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    P, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    PW, PT = ctypes.POINTER(QWeight), ctypes.POINTER(TT)
    lib.qa_version.restype = ctypes.c_char_p
    lib.qa_version.argtypes = []
    lib.qa_last_error.restype = ctypes.c_char_p
    lib.qa_last_error.argtypes = []
    lib.qa_quantize_rows.restype = I32
    lib.qa_quantize_rows.argtypes = [P, I32, I64, I64, I64, I32, P, I64, I64, P, P, P, P, P]
    lib.qa_dequantize_rows.restype = I32
    lib.qa_dequantize_rows.argtypes = [PW, P, I32, I64, I32, P]
    lib.qa_qmatmul_workspace_bytes.restype = SZ
    lib.qa_qmatmul_workspace_bytes.argtypes = [PW, I64, I32]
    lib.qa_qmatmul.restype = I32
    lib.qa_qmatmul.argtypes = [PW, P, I32, I64, P, P, SZ, P]
    lib.qa_qmatmul_t.restype = I32
    lib.qa_qmatmul_t.argtypes = [PW, P, I32, I64, P, P, SZ, P]
    lib.qa_code_rowsum.restype = I32
    lib.qa_code_rowsum.argtypes = [P, I64, I64, I32, P, P]
    F32 = ctypes.c_float
    lib.qa_rmsnorm_forward.restype = I32
    lib.qa_rmsnorm_forward.argtypes = [P, P, P, P, I64, I64, F32, P, P, P]
    lib.qa_rmsnorm_backward.restype = I32
    lib.qa_rmsnorm_backward.argtypes = [P, P, P, I32, ctypes.POINTER(P), P, I64, I64, P, P]
    lib.qa_rope.restype = I32
    lib.qa_rope.argtypes = [P, P, I64, I64, I32, I32, P, P, I32, P]
    lib.qa_swiglu_forward.restype = I32
    lib.qa_swiglu_forward.argtypes = [P, P, P, I64, P]
    lib.qa_swiglu_backward.restype = I32
    lib.qa_swiglu_backward.argtypes = [P, P, P, P, P, I64, P]
    lib.qa_cross_entropy.restype = I32
    lib.qa_cross_entropy.argtypes = [P, P, I64, I64, P, P, P]
    lib.qa_mse.restype = I32
    lib.qa_mse.argtypes = [P, I32, P, I64, I64, P, P, I32, P]
    lib.qa_linear_workspace_bytes.restype = SZ
    lib.qa_linear_workspace_bytes.argtypes = [PW, PT, I64]
    lib.qa_linear_forward.restype = I32
    lib.qa_linear_forward.argtypes = [PW, PT, P, I32, I64, P, P, P, P, P, SZ, P]
    lib.qa_linear_backward.restype = I32
    lib.qa_linear_backward.argtypes = [PW, PT, P, I32, P, I32, I64, P, P, ctypes.POINTER(P), I32, P, SZ, P]
    lib.qa_linear_saved_bytes.restype = SZ
    lib.qa_linear_saved_bytes.argtypes = [PW, PT, I64]
    lib.qa_linear_forward_save.restype = I32
    lib.qa_linear_forward_save.argtypes = [PW, PT, P, I32, I64, P, P, SZ, P, SZ, P]
    lib.qa_linear_backward_saved.restype = I32
    lib.qa_linear_backward_saved.argtypes = [PW, PT, P, I32, P, I32, I64, P, ctypes.POINTER(P), I32, P, SZ, P, SZ, P]
    PP = ctypes.POINTER(P)
    lib.qa_group_workspace_bytes.restype = SZ
    lib.qa_group_workspace_bytes.argtypes = [I32, ctypes.POINTER(PW), ctypes.POINTER(PT), I64]
    lib.qa_group_forward.restype = I32
    lib.qa_group_forward.argtypes = [I32, ctypes.POINTER(PW), ctypes.POINTER(PT), P, I32, I64, PP, PP,
                                     ctypes.POINTER(SZ), P, SZ, P]
    lib.qa_group_backward.restype = I32
    lib.qa_group_backward.argtypes = [I32, ctypes.POINTER(PW), ctypes.POINTER(PT), P, I32, PP, I32, I64, PP,
                                      ctypes.POINTER(PP), I32, PP, ctypes.POINTER(SZ), P, SZ, P]
    D = ctypes.c_double
    lib.qa_adamw_step.restype = I32
    lib.qa_adamw_step.argtypes = [P, P, P, P, P, I64, D, D, D, D, D, I64, P]
    lib.qa_nonfinite_segments.restype = I32
    lib.qa_nonfinite_segments.argtypes = [P, P, I32, P, P]
    lib.qa_merge_workspace_bytes.restype = SZ
    lib.qa_merge_workspace_bytes.argtypes = [PT]
    lib.qa_merge.restype = I32
    lib.qa_merge.argtypes = [PW, PT, P, I32, P, SZ, P]
    lib.qa_tt_materialize.restype = I32
    lib.qa_tt_materialize.argtypes = [PT, P, P, SZ, P]
    lib.qa_gemm_bf16.restype = I32
    lib.qa_gemm_bf16.argtypes = [P, I64, P, I64, I64, I64, I64, P, P, I64, P]
    lib.qa_launch_count.restype = I64
    lib.qa_launch_count.argtypes = []
    lib.qa_timing_enable.restype = I32
    lib.qa_timing_enable.argtypes = [I32]
    lib.qa_timing_read.restype = I32
    lib.qa_timing_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64),
                                   ctypes.POINTER(ctypes.c_double)]
    return lib


def lib():
    """The loaded library (built on first use if the source is newer)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if "QADAPTER_LIB" not in os.environ:
                from . import build as _build

                try:
                    _build.build()
                except Exception as exc:  # pragma: no cover - surfaced loudly below
                    if not os.path.exists(LIB_PATH):
                        raise RuntimeError(f"libqadapter.so missing and build failed: {exc}") from exc
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libqadapter.so not found at {LIB_PATH}; run __graft_entry__.build()")
            _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


def timing_read(kernel_class: str):
    """(total_ms, launches, algorithmic work) recorded for a kernel class since qa_timing_enable(1)."""
    ms, n, w = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
    check(lib().qa_timing_read(kernel_class.encode(), ctypes.byref(ms), ctypes.byref(n), ctypes.byref(w)),
          "qa_timing_read")
    return ms.value, n.value, w.value


class QAError(RuntimeError):
    pass


def check(status: int, what: str):
    """Map a qa_status to the reference's exception classes (quant.QuantError / ModelError)."""
    if status == QA_OK:
        return
    msg = f"{what}: {lib().qa_last_error().decode(errors='replace')}"
    from .quant import QuantError
    from .linear import ModelError

    if status == QA_ERR_BITS:
        raise QuantError(msg)
    if status == QA_ERR_ARG:
        raise ModelError(msg)
    raise QAError(f"{msg} (status {status})")
