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


def qmatmul(q: QuantizedMatrix, x) -> torch.Tensor:
    """quant.py:123-132 as the paper computes it: x is quantised per token to 8 bits,
    multiplied with the codes on int8 tensor cores and dequantised in the epilogue.
    x: (..., cols) float32 / bfloat16 -> (..., rows) in x's dtype."""
    from .linear import linear_forward

    return linear_forward(q, None, x)


def qmatmul_t(q: QuantizedMatrix, dy) -> torch.Tensor:
    """quant.py:135-144: dy (..., rows) -> dy·deq(W) (..., cols) on bf16 tensor cores."""
    from .linear import linear_backward

    return linear_backward(q, None, None, dy)[0]


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
