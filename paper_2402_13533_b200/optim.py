"""AdamW for the adapter parameters on the device (trainer.py:84-121), SURVEY §8(f) row 3.

`AdamWState` / `adamw_step` keep the reference's names and semantics: float64 masters and moments per
tensor (held here in one flat device buffer, tensors in sorted-name order), float32 working copies
rounded from the masters, tensors updated in sorted-name order, and `TrainError` naming the first
tensor whose gradient is non-finite (tensors before it in that order are updated, as in the reference
loop).  The update is `qa_adamw_step`, which replays the reference's float64 operation sequence, so
parameters and masters are bit-identical to the numpy optimizer (tests/test_gpu_optim.py).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .linear import params_changed
from .quant import _stream_ptr

__all__ = ["TrainError", "AdamWConfig", "AdamWState", "adamw_step"]


class TrainError(RuntimeError):
    """Same role as lrlm.trainer.TrainError."""


class AdamWConfig:
    """The optimizer fields of the reference's TrainConfig (trainer.py:58-64)."""

    def __init__(self, lr=3e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01):
        if not (0.0 < beta1 < 1.0 and 0.0 < beta2 < 1.0):
            raise TrainError("betas must lie in (0, 1)")
        if lr <= 0:
            raise TrainError("lr must be > 0")
        self.lr, self.beta1, self.beta2, self.eps, self.weight_decay = lr, beta1, beta2, eps, weight_decay


class AdamWState:
    """trainer.py:84-91: per-tensor m / v and float64 masters, as slices of flat device buffers."""

    def __init__(self, params: dict):
        self.step = 0
        self.names = sorted(params)
        dev = params[self.names[0]].data.device if self.names else torch.device("cuda")
        self.sizes = [params[k].data.numel() for k in self.names]
        self.offsets = [0]
        for n in self.sizes:
            self.offsets.append(self.offsets[-1] + n)
        total = self.offsets[-1]
        self.master = torch.cat([params[k].data.reshape(-1).to(torch.float64) for k in self.names]) \
            if self.names else torch.zeros(0, dtype=torch.float64, device=dev)
        self.m = torch.zeros(total, dtype=torch.float64, device=dev)
        self.v = torch.zeros(total, dtype=torch.float64, device=dev)
        self.flat = torch.empty(total, dtype=torch.float32, device=dev)  # working copies
        self.gflat = torch.empty(total, dtype=torch.float32, device=dev)
        self.seg = torch.tensor(self.offsets, dtype=torch.int64, device=dev)
        self.flags = torch.zeros(max(len(self.names), 1), dtype=torch.int32, device=dev)
        self.index = {k: i for i, k in enumerate(self.names)}

    def bind(self, params: dict) -> dict:
        """Make every parameter's data a view of the flat float32 working copy (values unchanged) and return
        name -> view of the flat gradient buffer.  A training loop that zeroes `gflat`, lets the backward
        accumulate into those views and calls adamw_step skips the per-tensor gather and copy-back."""
        self.flat.copy_(self.master.to(torch.float32))
        views = {}
        for k in self.names:
            i = self.index[k]
            a, b = self.offsets[i], self.offsets[i + 1]
            shape = params[k].data.shape
            params[k].data = self.flat[a:b].view(shape)
            views[k] = self.gflat[a:b].view(shape)
        return views

    def _is_view(self, t: torch.Tensor, base: torch.Tensor, i: int) -> bool:
        return (t.data_ptr() == base.data_ptr() + base.element_size() * self.offsets[i]
                and t.numel() == self.sizes[i] and t.is_contiguous())


def adamw_step(state: AdamWState, params: dict, grads: dict, config: AdamWConfig):
    """trainer.py:94-121 on the device."""
    state.step += 1
    names = sorted(grads)
    for k in names:
        if k not in state.index:
            raise TrainError(f"optimizer state missing for tensor {k}")
    if not names:
        return
    L = _lib.lib()
    dev = state.flat.device
    sp = _stream_ptr(dev)
    # gather the gradients into the flat buffer (tensors without a gradient keep a zero slice and are
    # not touched below); gradients that already are its slices (AdamWState.bind) need no copy
    for k in names:
        i = state.index[k]
        if not state._is_view(grads[k], state.gflat, i):
            state.gflat[state.offsets[i]:state.offsets[i + 1]].copy_(grads[k].reshape(-1).to(torch.float32))
    state.flags.zero_()
    _lib.check(L.qa_nonfinite_segments(state.gflat.data_ptr(), state.seg.data_ptr(), len(state.names),
                                       state.flags.data_ptr(), sp), "qa_nonfinite_segments")
    bad = state.flags.cpu()
    stop = None
    for k in names:
        if bad[state.index[k]]:
            stop = k
            break
    todo = names if stop is None else names[: names.index(stop)]
    # contiguous runs of the flat buffer, in sorted-name order
    runs, cur = [], None
    for k in todo:
        i = state.index[k]
        if cur is not None and cur[1] == state.offsets[i]:
            cur[1] = state.offsets[i + 1]
        else:
            cur = [state.offsets[i], state.offsets[i + 1]]
            runs.append(cur)
    for a, b in runs:
        _lib.check(L.qa_adamw_step(state.flat.data_ptr() + 4 * a, state.master.data_ptr() + 8 * a,
                                   state.m.data_ptr() + 8 * a, state.v.data_ptr() + 8 * a,
                                   state.gflat.data_ptr() + 4 * a, b - a, float(config.lr), float(config.beta1),
                                   float(config.beta2), float(config.eps), float(config.weight_decay),
                                   state.step, sp), "qa_adamw_step")
    if todo:
        params_changed()  # the kernels wrote the parameters through raw pointers
    for k in todo:
        i = state.index[k]
        p = params[k]
        if not state._is_view(p.data, state.flat, i):
            p.data.copy_(state.flat[state.offsets[i]:state.offsets[i + 1]].reshape(p.data.shape).to(p.data.dtype))
    if stop is not None:
        raise TrainError(f"non-finite gradient for tensor {stop}")
