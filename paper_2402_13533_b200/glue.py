"""Host wrappers of the decoder-layer glue entry points (include/qadapter.h, csrc/glue.cu): rmsnorm with the
residual add folded in and its backward (transformer.py:478-496), in-place rotary rotation (:506-519), SiLU
gating (:872-874) and the mean cross-entropy loss with its gradient (:569-588). bf16 activations, CUDA only —
every call goes through libqadapter.so and raises on a non-zero status."""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .quant import _stream_ptr

__all__ = ["rmsnorm", "rmsnorm_backward", "rope_", "swiglu", "swiglu_backward", "cross_entropy", "mse"]

RMSNORM_EPS = 1e-5  # transformer.py:53


def _bf16(t: torch.Tensor, name: str) -> torch.Tensor:
    if not (t.is_cuda and t.dtype == torch.bfloat16 and t.is_contiguous()):
        raise ValueError(f"{name}: expected a contiguous bf16 CUDA tensor, got {t.dtype} on {t.device}")
    return t


def rmsnorm(a, gain, b=None, eps: float = RMSNORM_EPS):
    """(y, inv) for s = a, or (y, inv, s) with s = bf16(a + b); a, b: [rows, dim] bf16, gain: [dim] f32."""
    _bf16(a, "rmsnorm input")
    rows, dim = a.shape
    y = torch.empty_like(a)
    inv = torch.empty(rows, dtype=torch.float32, device=a.device)
    s = torch.empty_like(a) if b is not None else None
    if b is not None:
        _bf16(b, "rmsnorm addend")
    _lib.check(_lib.lib().qa_rmsnorm_forward(a.data_ptr(), None if b is None else b.data_ptr(),
                                              None if s is None else s.data_ptr(), gain.data_ptr(), rows, dim, eps,
                                              y.data_ptr(), inv.data_ptr(), _stream_ptr(a.device)),
               "qa_rmsnorm_forward")
    return (y, inv) if b is None else (y, inv, s)


def rmsnorm_backward(x, gain, inv, dys, dres=None):
    """dx of the rmsnorm of x for the summed upstream gradients dys (1..3 tensors), plus dres if given."""
    _bf16(x, "rmsnorm_backward x")
    rows, dim = x.shape
    dys = [_bf16(d, "rmsnorm_backward dy") for d in dys]
    arr = (ctypes.c_void_p * len(dys))(*[d.data_ptr() for d in dys])
    dx = torch.empty_like(x)
    _lib.check(_lib.lib().qa_rmsnorm_backward(x.data_ptr(), gain.data_ptr(), inv.data_ptr(), len(dys), arr,
                                               None if dres is None else _bf16(dres, "dres").data_ptr(), rows, dim,
                                               dx.data_ptr(), _stream_ptr(x.device)), "qa_rmsnorm_backward")
    return dx


def rope_(q, k, cos, sin, heads: int, seq: int, inverse: bool = False):
    """Rotate q and k ([rows, dim] bf16, rows = batch * seq) in place; k may be None."""
    _bf16(q, "rope q")
    rows, dim = q.shape
    if k is not None:
        _bf16(k, "rope k")
    _lib.check(_lib.lib().qa_rope(q.data_ptr(), None if k is None else k.data_ptr(), rows, dim, dim // heads, seq,
                                  cos.data_ptr(), sin.data_ptr(), 1 if inverse else 0, _stream_ptr(q.device)),
               "qa_rope")
    return q, k


def swiglu(up, gate):
    act = torch.empty_like(_bf16(up, "swiglu up"))
    _lib.check(_lib.lib().qa_swiglu_forward(up.data_ptr(), _bf16(gate, "swiglu gate").data_ptr(), act.data_ptr(),
                                            up.numel(), _stream_ptr(up.device)), "qa_swiglu_forward")
    return act


def swiglu_backward(up, gate, dact):
    dup, dgate = torch.empty_like(up), torch.empty_like(gate)
    _lib.check(_lib.lib().qa_swiglu_backward(up.data_ptr(), gate.data_ptr(), _bf16(dact, "swiglu dact").data_ptr(),
                                             dup.data_ptr(), dgate.data_ptr(), up.numel(), _stream_ptr(up.device)),
               "qa_swiglu_backward")
    return dup, dgate


def cross_entropy(logits, targets):
    """(loss as a 0-d f32 tensor, dlogits bf16) for bf16 logits [rows, vocab] and int64 targets [rows]."""
    _bf16(logits, "cross_entropy logits")
    rows, vocab = logits.shape
    t = targets.reshape(-1).to(torch.int64).contiguous()
    if t.numel() != rows:
        raise IndexError(f"cross_entropy: {t.numel()} targets for {rows} rows of logits")
    if rows and not bool(((t >= 0) & (t < vocab)).all()):  # the reference indexes logits[row, target]
        raise IndexError(f"cross_entropy: target outside [0, {vocab})")
    loss_rows = torch.empty(rows, dtype=torch.float32, device=logits.device)
    dl = torch.empty_like(logits)
    _lib.check(_lib.lib().qa_cross_entropy(logits.data_ptr(), t.data_ptr(), rows, vocab, loss_rows.data_ptr(),
                                           dl.data_ptr(), _stream_ptr(logits.device)), "qa_cross_entropy")
    return loss_rows.mean(), dl


def mse(y, target, dy_dtype=None):
    """(loss as a 0-d f32 tensor, dL/dy) of L = mean (y - target)^2 over y [rows, cols] (f32 or
    bf16) and an f32 target of the same shape; dL/dy = 2 (y - target) / (rows * cols) in dy_dtype (y's dtype)."""
    from .quant import _dtype_code

    if tuple(y.shape) != tuple(target.shape):
        raise ValueError(f"mse: y {tuple(y.shape)} vs target {tuple(target.shape)}")
    y2 = y.reshape(-1, y.shape[-1]).contiguous()
    t2 = target.reshape(-1, y.shape[-1]).to(torch.float32).contiguous()
    rows, cols = y2.shape
    loss_rows = torch.empty(rows, dtype=torch.float32, device=y.device)
    dy = torch.empty(y2.shape, dtype=dy_dtype or y.dtype, device=y.device)
    _lib.check(_lib.lib().qa_mse(y2.data_ptr(), _dtype_code(y2), t2.data_ptr(), rows, cols, loss_rows.data_ptr(),
                                 dy.data_ptr(), _dtype_code(dy), _stream_ptr(y.device)), "qa_mse")
    return loss_rows.sum() / (rows * cols), dy.reshape(y.shape)
