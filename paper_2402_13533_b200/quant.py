"""Device mirror of the reference's quant.py (pkg/src/lrlm/quant.py).

Same names, argument meaning and error behaviour as the reference module; arrays are
torch CUDA tensors and every computation runs through libqadapter's sm_100a kernels.
Host numpy inputs are uploaded once; `QuantizedMatrix.to_numpy()` exports the exact
reference layout for parity checks and checkpoint I/O.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import QA_BF16, QA_F32

__all__ = [
    "QuantError",
    "QuantizedMatrix",
    "quantize_rows",
    "dequantize_rows",
    "qmatvec",
    "qmatmul",
    "qmatmul_t",
    "quantize_activations",
    "dequantize_activations",
    "quantized_size_bytes",
    "workspace",
]


class QuantError(ValueError):
    """Same role as lrlm.quant.QuantError (quant.py:28-29)."""


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return QA_F32
    if t.dtype == torch.bfloat16:
        return QA_BF16
    raise QuantError(f"unsupported dtype {t.dtype}; expected float32 or bfloat16")


def _as_device(a, device=None) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32)))
    if not t.is_cuda:
        t = t.to(device or "cuda", non_blocking=False)
    if t.dtype not in (torch.float32, torch.bfloat16):
        t = t.float()
    return t.contiguous()


class _Workspace:
    """Grow-only scratch buffer per (device, stream); the library never allocates."""

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int, device) -> torch.Tensor:
        dev = torch.device(device)
        key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
            self._bufs[key] = buf
        return buf


workspace = _Workspace()


@dataclass
class QuantizedMatrix:
    """quant.py:55-70 on the device: codes keep the reference layout (4-bit packed two per byte)."""

    rows: int
    cols: int
    bits: int
    codes: torch.Tensor  # uint8 [rows, cols] or [rows, ceil(cols/2)]
    scale: torch.Tensor  # float32 [rows]
    offset: torch.Tensor  # float32 [rows]
    rowsum: torch.Tensor  # int32 [rows], Σ codes (the GEMM epilogue term)

    def unpacked_codes(self) -> torch.Tensor:
        if self.bits == 4:
            out = torch.empty((self.rows, self.codes.shape[1] * 2), dtype=torch.uint8, device=self.codes.device)
            out[:, 0::2] = self.codes & 0x0F
            out[:, 1::2] = self.codes >> 4
            return out[:, : self.cols]
        return self.codes

    def nbytes(self) -> int:
        return self.codes.numel() + 4 * self.scale.numel() + 4 * self.offset.numel()

    @property
    def device(self):
        return self.codes.device

    def as_c(self) -> _lib.QWeight:
        return _lib.QWeight(self.rows, self.cols, self.bits, self.codes.data_ptr(), self.scale.data_ptr(),
                            self.offset.data_ptr(), self.rowsum.data_ptr())

    def to_numpy(self) -> dict:
        return {
            "codes": self.codes.cpu().numpy(),
            "scale": self.scale.cpu().numpy(),
            "offset": self.offset.cpu().numpy(),
        }


def quantize_rows(w, bits: int) -> QuantizedMatrix:
    """quant.py:73-99: per-row min/max codes, bit-exact with the reference."""
    if bits not in (4, 8):
        raise QuantError(f"bits must be 4 or 8, got {bits}")
    if isinstance(w, np.ndarray) or not isinstance(w, torch.Tensor):
        w = np.asarray(w)
        if w.ndim != 2:
            raise QuantError(f"expected 2-D grid, got shape {w.shape}")
    w = _as_device(w)
    if w.dim() != 2:
        raise QuantError(f"expected 2-D grid, got shape {tuple(w.shape)}")
    rows, cols = w.shape
    if rows == 0 or cols == 0:
        raise QuantError(f"cannot quantize an empty grid {tuple(w.shape)}")
    dev = w.device
    ld = cols if bits == 8 else (cols + 1) // 2
    codes = torch.empty((rows, ld), dtype=torch.uint8, device=dev)
    scale = torch.empty(rows, dtype=torch.float32, device=dev)
    offset = torch.empty(rows, dtype=torch.float32, device=dev)
    rowsum = torch.empty(rows, dtype=torch.int32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    st = _lib.lib().qa_quantize_rows(w.data_ptr(), _dtype_code(w), rows, cols, cols, bits, codes.data_ptr(), ld,
                                     cols, scale.data_ptr(), offset.data_ptr(), rowsum.data_ptr(), flag.data_ptr(),
                                     _stream_ptr(dev))
    _lib.check(st, "quantize_rows")
    if int(flag.item()) != 0:  # deferred device-side detection (quant.py:79-80)
        raise QuantError("cannot quantize non-finite values")
    return QuantizedMatrix(rows, cols, bits, codes, scale, offset, rowsum)


def dequantize_rows(q: QuantizedMatrix, dtype=torch.float32, transpose: bool = False) -> torch.Tensor:
    """quant.py:102-105: code·scale + offset in fp64, rounded to `dtype` (float32 or bfloat16)."""
    if dtype in (np.float32, "float32"):
        dtype = torch.float32
    shape = (q.cols, q.rows) if transpose else (q.rows, q.cols)
    out = torch.empty(shape, dtype=dtype, device=q.device)
    c = q.as_c()
    st = _lib.lib().qa_dequantize_rows(ctypes.byref(c), out.data_ptr(), _dtype_code(out), shape[1],
                                       1 if transpose else 0, _stream_ptr(q.device))
    _lib.check(st, "dequantize_rows")
    return out


def _flatten(x: torch.Tensor, k: int) -> torch.Tensor:
    if x.shape[-1] != k:
        raise QuantError(f"dimension mismatch: fan_in {k} vs x {tuple(x.shape)}")
    return x.reshape(-1, k).contiguous()


def _qmm(q: QuantizedMatrix, a: torch.Tensor, transpose: bool) -> torch.Tensor:
    """qa_qmatmul / qa_qmatmul_t on a contiguous 2-D float32 / bfloat16 operand."""
    T = a.shape[0]
    out = torch.empty((T, q.cols if transpose else q.rows), dtype=torch.float32, device=q.device)
    if T == 0:
        return out
    c = q.as_c()
    L = _lib.lib()
    ws = workspace.get(L.qa_qmatmul_workspace_bytes(ctypes.byref(c), T, 1 if transpose else 0), q.device)
    fn = L.qa_qmatmul_t if transpose else L.qa_qmatmul
    _lib.check(fn(ctypes.byref(c), a.data_ptr(), _dtype_code(a), T, out.data_ptr(), ws.data_ptr(), ws.numel(),
                  _stream_ptr(q.device)), "qmatmul_t" if transpose else "qmatmul")
    return out


def qmatvec(q: QuantizedMatrix, x) -> torch.Tensor:
    """quant.py:108-120: row i = scale_i (codes_i · x) + offset_i Σx, without dequantising (float32 result)."""
    x = _as_device(x, q.device)
    if x.shape[-1] != q.cols:
        raise QuantError(f"qmatvec dimension mismatch: {q.rows}x{q.cols} @ {tuple(x.shape)}")
    if x.dim() != 1:
        raise QuantError(f"qmatvec expects a 1-D vector, got shape {tuple(x.shape)}")
    return _qmm(q, x.reshape(1, -1), False)[0]


def qmatmul(q: QuantizedMatrix, x, act_quant: bool = False) -> torch.Tensor:
    """quant.py:123-132: x (..., cols) -> (..., rows) = (x·codesᵀ)·scale + Σx·offset (float32 result, the
    reference's fp64 formula to fp32 accuracy; qa_qmatmul).

    act_quant=True is the paper's forward instead: x quantised per token to 8 bits, an int8
    tensor-core GEMM and a dequantising epilogue (qa_linear_forward); the result then is in x's dtype."""
    if act_quant:
        from .linear import linear_forward

        return linear_forward(q, None, x)
    x = _as_device(x, q.device)
    if x.shape[-1] != q.cols:
        raise QuantError(f"qmatmul dimension mismatch: {q.rows}x{q.cols} vs {tuple(x.shape)}")
    lead = tuple(x.shape[:-1])
    return _qmm(q, x.reshape(-1, q.cols).contiguous(), False).reshape(*lead, q.rows)


def qmatmul_t(q: QuantizedMatrix, dy) -> torch.Tensor:
    """quant.py:135-144: dy (..., rows) -> dy·W = (dy·scale)·codes + dy·offset (float32 result, fp32-accurate;
    qa_qmatmul_t).  The training backward's bf16 path is QuantizedLinear.backward / linear_backward."""
    dy = _as_device(dy, q.device)
    if dy.shape[-1] != q.rows:
        raise QuantError(f"qmatmul_t dimension mismatch: {q.rows}x{q.cols} vs {tuple(dy.shape)}")
    lead = tuple(dy.shape[:-1])
    return _qmm(q, dy.reshape(-1, q.rows).contiguous(), True).reshape(*lead, q.cols)


def quantize_activations(x, bits: int) -> QuantizedMatrix:
    """quant.py:147-152: single-vector form of quantize_rows."""
    x = _as_device(x)
    if x.dim() != 1:
        raise QuantError(f"expected 1-D vector, got shape {tuple(x.shape)}")
    return quantize_rows(x[None, :], bits)


def dequantize_activations(q: QuantizedMatrix, dtype=torch.float32) -> torch.Tensor:
    return dequantize_rows(q, dtype)[0]


def quantized_size_bytes(param_count: int, bits: int, row_len: int) -> int:
    """quant.py:159-167 storage arithmetic (codes + two f32 per row for 4/8 bits)."""
    if param_count == 0:
        return 0
    if bits not in (4, 8, 16, 32):
        raise QuantError(f"unsupported bit width {bits}")
    code_bytes = -(-param_count * bits // 8)
    rows = -(-param_count // row_len)
    return code_bytes + (rows * 8 if bits in (4, 8) else 0)
