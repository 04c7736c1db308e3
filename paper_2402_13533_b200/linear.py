"""Device mirror of the reference's linear-backend protocol (pkg/src/lrlm/transformer.py:138-327)
and adapter lifecycle (pkg/src/lrlm/lowrank.py:189-281), with the paper's tensor-train adapter.

Backends keep the reference's duck-typed protocol: `kind`, `name`, `fan_in`, `fan_out`,
`params()`, `forward(x, step=0)`, `backward(x, dy, grads, step=0) -> dx`, `astype(dtype)`,
`merged`.  Gradients accumulate into the caller's dict exactly like `_accumulate`
(transformer.py:150-156): frozen tensors get no entry, repeated names add.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import QA_BF16, QA_F32
from .quant import QuantError, QuantizedMatrix, _as_device, _dtype_code, _stream_ptr, quantize_rows, workspace

__all__ = [
    "ModelError",
    "Param",
    "TTSpec",
    "QuantizedLinear",
    "TTLinear",
    "LoraLinear",
    "linear_forward",
    "linear_forward_saving",
    "linear_backward",
    "tt_materialize",
    "tt_merge",
    "lora_merge",
    "attach_tt_adapter",
    "group_forward",
    "group_backward",
]


class ModelError(ValueError):
    """Same role as lrlm.transformer.ModelError (transformer.py:61-62)."""


# Generation of the trainable parameters' values.  Kernels (the AdamW update, checkpoint loads) write
# parameters through raw pointers, which torch's _version counters never see; they bump this instead,
# so a recompute-window state saved before the update is not reused after it.
_param_generation = [0]


def params_changed() -> None:
    """Invalidate every saved recompute-window state (call after updating parameters in place)."""
    _param_generation[0] += 1


class Param:
    """transformer.py:138-147."""

    __slots__ = ("name", "data", "trainable")

    def __init__(self, name: str, data: torch.Tensor, trainable: bool = True):
        self.name = name
        self.data = data
        self.trainable = trainable

    def __repr__(self):
        return f"Param({self.name}, shape={tuple(self.data.shape)}, trainable={self.trainable})"


def _accumulate(grads: dict, param: Param, g: torch.Tensor):
    """transformer.py:150-156."""
    if not param.trainable:
        return
    if param.name in grads:
        grads[param.name] += g
    else:
        grads[param.name] = g


@dataclass(frozen=True)
class TTSpec:
    """Tensor-train adapter shape: core k is (ranks[k], m[k], n[k], ranks[k+1])."""

    m: tuple
    n: tuple
    ranks: tuple

    def __post_init__(self):
        if not 1 <= len(self.m) <= _lib.QA_TT_MAX_D or len(self.n) != len(self.m):
            raise ModelError(f"TT needs 1..{_lib.QA_TT_MAX_D} cores with matching modes")
        if len(self.ranks) != len(self.m) + 1 or self.ranks[0] != 1 or self.ranks[-1] != 1:
            raise ModelError("TT ranks must be (1, r_1, ..., r_{d-1}, 1)")

    @property
    def d(self) -> int:
        return len(self.m)

    @property
    def fan_out(self) -> int:
        return int(np.prod(self.m))

    @property
    def fan_in(self) -> int:
        return int(np.prod(self.n))

    def core_shape(self, k: int) -> tuple:
        return (self.ranks[k], self.m[k], self.n[k], self.ranks[k + 1])

    def param_count(self) -> int:
        return int(sum(np.prod(self.core_shape(k)) for k in range(self.d)))

    @staticmethod
    def for_shape(fan_out: int, fan_in: int, r: int) -> "TTSpec":
        """Pinned modes (DESIGN.md §TT modes): BASELINE config 1 is balanced (4,16,16)²;
        Llama shapes use m = (1, N/256, 256), n = (K/4, 4, 1): first core input-only, last core
        output-only, so every contraction touching x or dy has rank r on its small side."""
        if fan_out == 1024 and fan_in == 1024:
            return TTSpec((4, 16, 16), (4, 16, 16), (1, r, r, 1))
        if fan_out % 256 == 0 and fan_in % 4 == 0:
            return TTSpec((1, fan_out // 256, 256), (fan_in // 4, 4, 1), (1, r, r, 1))
        raise ModelError(f"no pinned TT modes for {fan_out}x{fan_in}; pass a TTSpec")

    @staticmethod
    def lora(fan_out: int, fan_in: int, r: int) -> "TTSpec":
        """LoRA ΔW = up·down as a 2-core TT: m = (1, N), n = (K, 1)."""
        return TTSpec((1, fan_out), (fan_in, 1), (1, r, 1))

    def as_c(self, cores) -> _lib.TT:
        tt = _lib.TT()
        tt.d = self.d
        for k in range(self.d):
            tt.m[k] = self.m[k]
            tt.n[k] = self.n[k]
            tt.cores[k] = cores[k].data_ptr()
        for k in range(self.d + 1):
            tt.r[k] = self.ranks[k]
        return tt


def _check_cores(spec: TTSpec, cores):
    if len(cores) != spec.d:
        raise ModelError(f"expected {spec.d} TT cores, got {len(cores)}")
    for k, c in enumerate(cores):
        if tuple(c.shape) != spec.core_shape(k) or c.dtype != torch.float32 or not c.is_cuda:
            raise ModelError(f"core {k}: expected cuda float32 {spec.core_shape(k)}, got {c.dtype} {tuple(c.shape)}")


def linear_forward(q: QuantizedMatrix, adapter, x, *, debug: bool = False):
    """y = deq(Q(x))·deq(Q(W))ᵀ + x·W_tᵀ through qa_linear_forward (adapter = (TTSpec, cores) or None).

    x: (..., fan_in) float32/bfloat16 -> (..., fan_out) in x's dtype.  debug=True returns a dict
    with the int32 accumulators, the fp32 y and the fp32 adapter term y2 as well."""
    x = _as_device(x, q.device)
    lead = tuple(x.shape[:-1])
    if x.shape[-1] != q.cols:
        raise QuantError(f"qmatmul dimension mismatch: {q.rows}x{q.cols} vs {tuple(x.shape)}")
    x2 = x.reshape(-1, q.cols).contiguous()
    T = x2.shape[0]
    dev = q.device
    y = torch.empty((T, q.rows), dtype=torch.bfloat16, device=dev)
    want_f32 = debug or x2.dtype == torch.float32
    y32 = torch.empty((T, q.rows), dtype=torch.float32, device=dev) if want_f32 else None
    acc = torch.empty((T, q.rows), dtype=torch.int32, device=dev) if debug else None
    y2 = torch.empty((T, q.rows), dtype=torch.float32, device=dev) if (debug and adapter is not None) else None
    wc = q.as_c()
    ttc = None
    if adapter is not None:
        spec, cores = adapter
        _check_cores(spec, cores)
        ttc = spec.as_c(cores)
    L = _lib.lib()
    nbytes = L.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc) if ttc else None, T)
    if nbytes == 0:
        raise ModelError(f"invalid linear configuration: {L.qa_last_error().decode()}")
    ws = workspace.get(nbytes, dev)
    st = L.qa_linear_forward(ctypes.byref(wc), ctypes.byref(ttc) if ttc else None, x2.data_ptr(), _dtype_code(x2), T,
                             y.data_ptr(), acc.data_ptr() if acc is not None else None,
                             y32.data_ptr() if y32 is not None else None,
                             y2.data_ptr() if y2 is not None else None, ws.data_ptr(), ws.numel(), _stream_ptr(dev))
    _lib.check(st, "qa_linear_forward")
    out = (y32 if x2.dtype == torch.float32 else y).reshape(*lead, q.rows)
    if not debug:
        return out
    return {"y": out, "y_bf16": y.reshape(*lead, q.rows), "y_f32": y32.reshape(*lead, q.rows),
            "acc": acc.reshape(*lead, q.rows), "y2": None if y2 is None else y2.reshape(*lead, q.rows)}


def linear_forward_saving(q: QuantizedMatrix, adapter, x):
    """Forward of the recompute window (qa_linear_forward_save): returns (y, saved), where `saved`
    is the adapter state the backward of the SAME x and cores can take instead of re-reading x
    (the fast TT family's Z1; None when the adapter has nothing to save)."""
    x = _as_device(x, q.device)
    lead = tuple(x.shape[:-1])
    if x.shape[-1] != q.cols:
        raise QuantError(f"qmatmul dimension mismatch: {q.rows}x{q.cols} vs {tuple(x.shape)}")
    x2 = x.reshape(-1, q.cols).contiguous()
    if adapter is None or x2.dtype != torch.bfloat16:
        return linear_forward(q, adapter, x), None
    T = x2.shape[0]
    dev = q.device
    spec, cores = adapter
    _check_cores(spec, cores)
    wc, ttc = q.as_c(), spec.as_c(cores)
    L = _lib.lib()
    nsaved = L.qa_linear_saved_bytes(ctypes.byref(wc), ctypes.byref(ttc), T)
    if nsaved == 0:
        return linear_forward(q, adapter, x), None
    saved = torch.empty(nsaved // 4, dtype=torch.float32, device=dev)
    y = torch.empty((T, q.rows), dtype=torch.bfloat16, device=dev)
    nbytes = L.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc), T)
    ws = workspace.get(nbytes, dev)
    _lib.check(L.qa_linear_forward_save(ctypes.byref(wc), ctypes.byref(ttc), x2.data_ptr(), _dtype_code(x2), T,
                                        y.data_ptr(), saved.data_ptr(), nsaved, ws.data_ptr(), ws.numel(),
                                        _stream_ptr(dev)), "qa_linear_forward_save")
    return y.reshape(*lead, q.rows), saved


def linear_backward(q: QuantizedMatrix, adapter, x, dy, *, want_dx: bool = True, want_grads: bool = True,
                    debug: bool = False, saved: torch.Tensor | None = None, grad_out=None):
    """dx = dy·deq(W) + dy·W_t and the adapter-core gradients through qa_linear_backward.

    grad_out: float32 tensors shaped like the cores; the gradients are then added into them in the kernels
    (the C ABI's accumulate flag) and None is returned in their place.
    Returns (dx or None, [dG_k] or None[, dx_f32 when debug])."""
    dy = _as_device(dy, q.device)
    lead = tuple(dy.shape[:-1])
    if dy.shape[-1] != q.rows:
        raise QuantError(f"qmatmul_t dimension mismatch: {q.rows}x{q.cols} vs {tuple(dy.shape)}")
    dy2 = dy.reshape(-1, q.rows).contiguous()
    T = dy2.shape[0]
    dev = q.device
    x2 = None
    if adapter is not None:
        x = _as_device(x, dev)
        x2 = x.reshape(-1, q.cols).contiguous()
        if x2.shape[0] != T:
            raise ModelError(f"x has {x2.shape[0]} tokens but dy has {T}")
    dx = torch.empty((T, q.cols), dtype=torch.bfloat16, device=dev) if want_dx else None
    dx32 = torch.empty((T, q.cols), dtype=torch.float32, device=dev) if (want_dx and (debug or dy2.dtype == torch.float32)) else None
    wc = q.as_c()
    ttc, grads, gptrs = None, None, None
    if adapter is not None:
        spec, cores = adapter
        _check_cores(spec, cores)
        ttc = spec.as_c(cores)
        if want_grads:
            grads = grad_out if grad_out is not None else \
                [torch.empty(spec.core_shape(k), dtype=torch.float32, device=dev) for k in range(spec.d)]
            gptrs = (ctypes.c_void_p * _lib.QA_TT_MAX_D)(*[g.data_ptr() for g in grads])
    accumulate = 1 if (grad_out is not None and grads is not None) else 0
    L = _lib.lib()
    nbytes = L.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc) if ttc else None, T)
    if nbytes == 0:
        raise ModelError(f"invalid linear configuration: {L.qa_last_error().decode()}")
    ws = workspace.get(nbytes, dev)
    if saved is not None and ttc is not None and dx32 is None:
        st = L.qa_linear_backward_saved(ctypes.byref(wc), ctypes.byref(ttc), x2.data_ptr(), _dtype_code(x2),
                                        dy2.data_ptr(), _dtype_code(dy2), T,
                                        dx.data_ptr() if dx is not None else None,
                                        ctypes.cast(gptrs, ctypes.POINTER(ctypes.c_void_p)) if gptrs is not None
                                        else None, accumulate, saved.data_ptr(), saved.numel() * 4, ws.data_ptr(),
                                        ws.numel(), _stream_ptr(dev))
        _lib.check(st, "qa_linear_backward_saved")
        out_dx = None if dx is None else dx.reshape(*lead, q.cols)
        grads = None if accumulate else grads
        return (out_dx, grads, None) if debug else (out_dx, grads)
    st = L.qa_linear_backward(ctypes.byref(wc), ctypes.byref(ttc) if ttc else None,
                              x2.data_ptr() if x2 is not None else None,
                              _dtype_code(x2) if x2 is not None else QA_F32, dy2.data_ptr(), _dtype_code(dy2), T,
                              dx.data_ptr() if dx is not None else None,
                              dx32.data_ptr() if dx32 is not None else None,
                              ctypes.cast(gptrs, ctypes.POINTER(ctypes.c_void_p)) if gptrs is not None else None,
                              accumulate, ws.data_ptr(), ws.numel(), _stream_ptr(dev))
    _lib.check(st, "qa_linear_backward")
    grads = None if accumulate else grads
    out_dx = None
    if want_dx:
        out_dx = (dx32 if dy2.dtype == torch.float32 else dx).reshape(*lead, q.cols)
    if debug:
        return out_dx, grads, None if dx32 is None else dx32.reshape(*lead, q.cols)
    return out_dx, grads


def tt_materialize(spec: TTSpec, cores) -> torch.Tensor:
    """W_t [fan_out, fan_in] fp32: the contraction of the cores."""
    _check_cores(spec, cores)
    dev = cores[0].device
    ttc = spec.as_c(cores)
    L = _lib.lib()
    nb = L.qa_merge_workspace_bytes(ctypes.byref(ttc))
    ws = workspace.get(nb, dev)
    out = torch.empty((spec.fan_out, spec.fan_in), dtype=torch.float32, device=dev)
    _lib.check(L.qa_tt_materialize(ctypes.byref(ttc), out.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(dev)),
               "qa_tt_materialize")
    return out


def _merge(q: QuantizedMatrix, spec: TTSpec, cores, dtype) -> torch.Tensor:
    _check_cores(spec, cores)
    dev = q.device
    wc, ttc = q.as_c(), spec.as_c(cores)
    L = _lib.lib()
    nb = L.qa_merge_workspace_bytes(ctypes.byref(ttc))
    ws = workspace.get(nb, dev)
    out = torch.empty((q.rows, q.cols), dtype=dtype, device=dev)
    _lib.check(L.qa_merge(ctypes.byref(wc), ctypes.byref(ttc), out.data_ptr(), _dtype_code(out), ws.data_ptr(),
                          ws.numel(), _stream_ptr(dev)), "qa_merge")
    return out


def _dense_forward(w_bf16: torch.Tensor, x) -> torch.Tensor:
    """Merged inference path: y = x·W'ᵀ on bf16 tensor cores (qa_gemm_bf16)."""
    x = _as_device(x, w_bf16.device)
    lead = tuple(x.shape[:-1])
    n, k = w_bf16.shape
    x2 = x.reshape(-1, k).to(torch.bfloat16).contiguous()
    T = x2.shape[0]
    y32 = torch.empty((T, n), dtype=torch.float32, device=w_bf16.device)
    _lib.check(_lib.lib().qa_gemm_bf16(x2.data_ptr(), k, w_bf16.data_ptr(), k, T, n, k, None, y32.data_ptr(), n,
                                       _stream_ptr(w_bf16.device)), "qa_gemm_bf16")
    return y32.to(x.dtype).reshape(*lead, n)


class QuantizedLinear:
    """transformer.py:246-273: frozen quantised base; forward = qmatmul, backward = qmatmul_t."""

    kind = "quantized"

    def __init__(self, name: str, q: QuantizedMatrix):
        self.name = name
        self.q = q

    @property
    def fan_out(self):
        return self.q.rows

    @property
    def fan_in(self):
        return self.q.cols

    def params(self):
        return []

    def forward(self, x, step: int = 0):
        return linear_forward(self.q, None, x)

    def backward(self, x, dy, grads, step: int = 0):
        return linear_backward(self.q, None, None, dy, want_grads=False)[0]

    def astype(self, dtype):
        return self


class TTLinear:
    """The paper's layer: frozen quantised base + trainable tensor-train adapter.

    forward  : y = deq(Q(x))·deq(Q(W))ᵀ + x·W_tᵀ   (one fused qa_linear_forward)
    backward : recomputes the TT partial contractions from the stored input x, accumulates the
               core gradients, returns dx (LoraLinear.backward semantics, transformer.py:310-318)
    merge    : W' = dequantize_rows(q) + W_t       (tt_merge)
    """

    kind = "tt"

    def __init__(self, name: str, base: QuantizedLinear, spec: TTSpec, cores):
        if not isinstance(base, QuantizedLinear):
            raise ModelError(f"{name}: adapters need a quantized base, found {getattr(base, 'kind', type(base))}")
        if spec.fan_out != base.fan_out or spec.fan_in != base.fan_in:
            raise ModelError(f"{name}: TT modes {spec.fan_out}x{spec.fan_in} do not match the base "
                             f"{base.fan_out}x{base.fan_in}")
        self.name = name
        self.base = base
        self.spec = spec
        self.cores = [Param(f"{name}.core{k}", c, True) for k, c in enumerate(cores)]
        _check_cores(spec, [p.data for p in self.cores])
        self.merged = False
        self._merged_weight = None
        self._merged_bf16 = None

    @property
    def fan_out(self):
        return self.base.fan_out

    @property
    def fan_in(self):
        return self.base.fan_in

    def params(self):
        return self.base.params() + list(self.cores)

    def _core_tensors(self):
        return [p.data.contiguous() for p in self.cores]

    def _scatter_grads(self, grads: dict, dcores):
        for p, g in zip(self.cores, dcores):
            _accumulate(grads, p, g)

    def _grad_dest(self, grads: dict):
        """Preallocated float32 gradient buffers for every core (e.g. views of an optimizer's flat gradient
        buffer), or None: then the kernels accumulate into them directly instead of returning new tensors."""
        out = []
        for p in self.cores:
            g = grads.get(p.name)
            if not p.trainable or not (isinstance(g, torch.Tensor) and g.is_cuda and g.dtype == torch.float32 and
                                       g.is_contiguous() and g.shape == p.data.shape):
                return None
            out.append(g)
        return out if out else None

    def _tag(self, x):
        return (x.data_ptr(), tuple(x.shape), x._version, _param_generation[0],
                tuple(p.data._version for p in self._params_for_tag()))

    def _params_for_tag(self):
        return self.cores

    def forward(self, x, step: int = 0):
        """y = base(x) + adapter(x).  When x is a bf16 CUDA tensor the recompute-window state
        (Z1, qa_linear_forward_save) is kept for a following backward on the same, unmodified x
        and cores — the PER_LAYER pattern of re-running a layer's forward right before its
        backward (transformer.py:888-897); any other backward recomputes it from x."""
        if self.merged:
            return _dense_forward(self._merged_bf16, x)
        self._saved = None
        if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.bfloat16:
            y, saved = linear_forward_saving(self.base.q, (self.spec, self._core_tensors()), x)
            if saved is not None:
                self._saved = (weakref.ref(x), self._tag(x), saved)
            return y
        return linear_forward(self.base.q, (self.spec, self._core_tensors()), x)

    def _take_saved(self, x):
        s, self._saved = getattr(self, "_saved", None), None
        if s is None or not isinstance(x, torch.Tensor):
            return None
        ref, tag, saved = s
        return saved if ref() is x and self._tag(x) == tag else None

    def backward(self, x, dy, grads, step: int = 0):
        if self.merged:
            raise ModelError(f"{self.name}: merged adapter is inference-only")
        saved = self._take_saved(x)
        dest = self._grad_dest(grads)
        dx, dcores = linear_backward(self.base.q, (self.spec, self._core_tensors()), x, dy, saved=saved,
                                     grad_out=dest)
        if dest is None:
            self._scatter_grads(grads, dcores)
        return dx

    def astype(self, dtype):
        return self


class LoraLinear(TTLinear):
    """transformer.py:276-327 over a QuantizedLinear base: ΔW = up·down, run as the 2-core TT
    m = (1, N), n = (K, 1) so it shares every kernel with the tensor adapter."""

    kind = "lora"

    def __init__(self, name: str, base: QuantizedLinear, down, up):
        down = _as_device(down, base.q.device).float()
        up = _as_device(up, base.q.device).float()
        if down.shape[0] != up.shape[1]:
            raise ModelError(f"{name}: rank mismatch {tuple(down.shape)} vs {tuple(up.shape)}")
        r = down.shape[0]
        self.down = Param(name + ".down", down, True)
        self.up = Param(name + ".up", up, True)
        spec = TTSpec.lora(up.shape[0], down.shape[1], r)
        TTLinear.__init__(self, name, base, spec, self._lora_cores(down, up))
        self.cores = []  # the trainable tensors are .down / .up

    @staticmethod
    def _lora_cores(down, up):
        r, k = down.shape
        n = up.shape[0]
        return [down.t().contiguous().reshape(1, 1, k, r), up.t().contiguous().reshape(r, n, 1, 1)]

    @property
    def rank(self):
        return self.down.data.shape[0]

    def _params_for_tag(self):
        return [self.down, self.up]

    def params(self):
        return self.base.params() + [self.down, self.up]

    def _core_tensors(self):
        return self._lora_cores(self.down.data, self.up.data)

    def _grad_dest(self, grads: dict):
        return None  # the trainable tensors are .down / .up (transposed cores)

    def _scatter_grads(self, grads: dict, dcores):
        r, k = self.down.data.shape
        n = self.up.data.shape[0]
        _accumulate(grads, self.down, dcores[0].reshape(k, r).t().contiguous())
        _accumulate(grads, self.up, dcores[1].reshape(r, n).t().contiguous())


def tt_merge(adapter: TTLinear, dtype=torch.float32) -> torch.Tensor:
    """lowrank.lora_merge (lowrank.py:245-257) for a quantised base, through the explicit
    dequantise route its error message prescribes (lowrank.py:249-252): W' = deq(q) + W_t."""
    if adapter.merged:
        raise ModelError(f"{adapter.name}: adapter already merged")
    merged = _merge(adapter.base.q, adapter.spec, adapter._core_tensors(), dtype)
    adapter.merged = True
    adapter._merged_weight = merged
    adapter._merged_bf16 = merged.to(torch.bfloat16).contiguous()
    return merged


lora_merge = tt_merge


def attach_tt_adapter(name: str, base: QuantizedLinear, r: int, spec: TTSpec | None = None, seed: int = 0,
                      std: float = 0.01, zero_last: bool = False) -> TTLinear:
    """attach_adapters (lowrank.py:189-234) for one matrix: cores ~N(0, std²) from a seeded
    generator; zero_last=True zeroes the last core so the adapter starts as the identity delta."""
    spec = spec or TTSpec.for_shape(base.fan_out, base.fan_in, r)
    if any(rk >= min(base.fan_in, base.fan_out) for rk in spec.ranks[1:-1]):
        raise ModelError(f"{name}: rank must be < min(fan_in, fan_out)")
    gen = torch.Generator(device=base.q.device).manual_seed(int(seed))
    cores = []
    for k in range(spec.d):
        c = torch.randn(spec.core_shape(k), generator=gen, device=base.q.device, dtype=torch.float32) * std
        if zero_last and k == spec.d - 1:
            c.zero_()
        cores.append(c)
    return TTLinear(name, base, spec, cores)


def quantized_linear(name: str, w, bits: int) -> QuantizedLinear:
    """quantize_model's per-matrix conversion (transformer.py:1122-1127)."""
    return QuantizedLinear(name, quantize_rows(w, bits))


# ------------------------------------------------------------------------ shared-input groups
def _group_c(members):
    """ctypes arrays for qa_group_*; the returned tuple keeps every referenced object alive."""
    n = len(members)
    cores = [m._core_tensors() for m in members]
    wcs = [m.base.q.as_c() for m in members]
    tts = [m.spec.as_c(c) for m, c in zip(members, cores)]
    W = (ctypes.POINTER(_lib.QWeight) * n)(*[ctypes.pointer(w) for w in wcs])
    Tt = (ctypes.POINTER(_lib.TT) * n)(*[ctypes.pointer(t) for t in tts])
    return W, Tt, (cores, wcs, tts)


def group_forward(members, x, step: int = 0):
    """Forward of members that read the same input (a decoder layer's wq / wk / wv on norm1 or
    wu / wg on norm2, transformer.py:862-874) through qa_group_forward: the act-quant codes and
    every member's Z1 come from one pass over x.  Returns [y_i]; each member keeps its
    recompute-window state for a following backward on the same x (TTLinear.forward)."""
    if not members:
        return []
    if any(not isinstance(m, TTLinear) or m.merged for m in members) or len(members) > 3:
        return [m.forward(x, step) for m in members]
    q0 = members[0].base.q
    x = _as_device(x, q0.device)
    lead = tuple(x.shape[:-1])
    x2 = x.reshape(-1, q0.cols).contiguous()
    if x2.dtype != torch.bfloat16 or any(m.fan_in != q0.cols for m in members):
        return [m.forward(x, step) for m in members]
    T, dev, n = x2.shape[0], q0.device, len(members)
    W, Tt, keep = _group_c(members)
    L = _lib.lib()
    ys = [torch.empty((T, m.fan_out), dtype=torch.bfloat16, device=dev) for m in members]
    nsv = [L.qa_linear_saved_bytes(ctypes.byref(keep[1][i]), ctypes.byref(keep[2][i]), T) for i in range(n)]
    saved = [torch.empty(max(b, 4) // 4, dtype=torch.float32, device=dev) for b in nsv]
    nb = L.qa_group_workspace_bytes(n, W, Tt, T)
    if nb == 0:
        raise ModelError(f"invalid group: {L.qa_last_error().decode()}")
    ws = workspace.get(nb, dev)
    Y = (ctypes.c_void_p * n)(*[y.data_ptr() for y in ys])
    S = (ctypes.c_void_p * n)(*[sv.data_ptr() if b else None for sv, b in zip(saved, nsv)])
    SB = (ctypes.c_size_t * n)(*nsv)
    _lib.check(L.qa_group_forward(n, W, Tt, x2.data_ptr(), QA_BF16, T, Y, S, SB, ws.data_ptr(), ws.numel(),
                                  _stream_ptr(dev)), "qa_group_forward")
    for m, sv, b in zip(members, saved, nsv):
        m._saved = (weakref.ref(x), m._tag(x), sv) if b else None
    return [y.reshape(*lead, y.shape[-1]) for y in ys]


def group_backward(members, x, dys, grads: dict, step: int = 0):
    """Backward of a shared-input group (transformer.py:919-944) through qa_group_backward: one
    pass over x for every member's dG1.  Accumulates the core gradients into `grads` like
    _accumulate and returns [dx_i] (the caller sums them, as _layer_backward does)."""
    if not members:
        return []
    simple = any(not isinstance(m, TTLinear) or m.merged or isinstance(m, LoraLinear) for m in members)
    q0 = members[0].base.q if not simple else None
    if simple or len(members) > 3:
        return [m.backward(x, dy, grads, step) for m, dy in zip(members, dys)]
    x = _as_device(x, q0.device)
    lead = tuple(x.shape[:-1])
    x2 = x.reshape(-1, q0.cols).contiguous()
    dys2 = [_as_device(dy, q0.device).reshape(-1, m.fan_out).contiguous() for m, dy in zip(members, dys)]
    T, dev, n = x2.shape[0], q0.device, len(members)
    W, Tt, keep = _group_c(members)
    L = _lib.lib()
    savedl = [m._take_saved(x) for m in members]
    dxs = [torch.empty((T, q0.cols), dtype=torch.bfloat16, device=dev) for _ in members]
    dests = [m._grad_dest(grads) for m in members]
    accumulate = 1 if all(d is not None for d in dests) else 0
    gr = dests if accumulate else \
        [[torch.empty(m.spec.core_shape(k), dtype=torch.float32, device=dev) for k in range(m.spec.d)]
         for m in members]
    nb = L.qa_group_workspace_bytes(n, W, Tt, T)
    if nb == 0:
        raise ModelError(f"invalid group: {L.qa_last_error().decode()}")
    ws = workspace.get(nb, dev)
    DY = (ctypes.c_void_p * n)(*[d.data_ptr() for d in dys2])
    DX = (ctypes.c_void_p * n)(*[d.data_ptr() for d in dxs])
    per = [(ctypes.c_void_p * _lib.QA_TT_MAX_D)(*[g.data_ptr() for g in gm]) for gm in gr]
    DC = (ctypes.POINTER(ctypes.c_void_p) * n)(*[ctypes.cast(p, ctypes.POINTER(ctypes.c_void_p)) for p in per])
    S = (ctypes.c_void_p * n)(*[sv.data_ptr() if sv is not None else None for sv in savedl])
    SB = (ctypes.c_size_t * n)(*[sv.numel() * 4 if sv is not None else 0 for sv in savedl])
    dy_dtype = _dtype_code(dys2[0])
    _lib.check(L.qa_group_backward(n, W, Tt, x2.data_ptr(), _dtype_code(x2), DY, dy_dtype, T, DX, DC, accumulate, S,
                                   SB, ws.data_ptr(), ws.numel(), _stream_ptr(dev)), "qa_group_backward")
    if not accumulate:
        for m, g in zip(members, gr):
            m._scatter_grads(grads, g)
    return [d.reshape(*lead, q0.cols) for d in dxs]
