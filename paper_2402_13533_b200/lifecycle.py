"""Adapter lifecycle over whole models and the host-side drop-in for the reference's numpy models.

The reference drives its linears through a duck-typed protocol on numpy arrays (transformer.py:174-391) from
`model_forward` / `model_backward` / `kv_decode_step` / `greedy_decode` (transformer.py:949-1111), and manages
adapters per model with `quantize_model` (transformer.py:1114-1139), `attach_adapters` / `merge_model`
(lowrank.py:189-281) and `configure_trainable` (trainer.py:124-151).  This module gives those model-level
functions for the device backends and `HostLinear`, the numpy <-> device shim that lets a reference
`DecoderModel` run its own forward / backward / decode loops with every quantised linear on the B200:

    model = lrlm.transformer.build_model(cfg, seed=0)               # the reference's model object
    model = lifecycle.quantize_model(model, 8)                       # device codes (bit-exact quantize_rows)
    model = lifecycle.attach_adapters(model, r=8, targets=(...))      # device LoRA (or kind="tt") adapters
    lifecycle.configure_trainable(model, "lora_finetune")
    logits, tape = lrlm.transformer.model_forward(model, tokens, lrlm.transformer.PER_LAYER)   # unchanged

Two semantics per backend:
  act_quant=True  (default): the paper's layer: x quantised per token, int8 tcgen05 GEMM with
                  the adapter folded in — the B200 hot path;
  act_quant=False : the reference's own arithmetic (qmatmul / qmatmul_t without activation quantisation,
                  quant.py:123-144) to fp32 accuracy, plus the adapter — a drop-in whose results match the
                  reference's CPU run.
The model objects themselves are the caller's classes (reference DecoderModel / DecoderLayer, duck-typed:
`layers[i].matrices()`, `layers[i].index / norm1 / norm2`, `head`, `config`, `specs`, `embed`, `dtype`); this
module never imports the reference package.
"""

from __future__ import annotations

import numpy as np
import torch

from .linear import LoraLinear, ModelError, Param, QuantizedLinear, TTLinear, TTSpec, _accumulate, linear_backward, \
    linear_forward, tt_merge
from .quant import QuantizedMatrix, qmatmul, qmatmul_t, quantize_rows

__all__ = ["HostLinear", "MATRIX_NAMES", "to_device", "quantize_model", "attach_adapters", "configure_trainable",
           "merge_model", "seeded_gaussian"]

MATRIX_NAMES = ("wq", "wk", "wv", "wo", "wu", "wg", "wd", "we", "wh")  # transformer.py:56
LAYER_MATS = ("wq", "wk", "wv", "wo", "wu", "wg", "wd")
INIT_STD = 0.02  # transformer.py INIT_STD, lowrank.py:221-223


# --------------------------------------------------------------------------- seeded factors
_GAMMA, _M1, _M2 = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def seeded_gaussian(rows: int, cols: int, seed: int, std: float = 1.0, dtype=np.float32) -> np.ndarray:
    """linalg.seeded_random(rows, cols, seed, "gaussian", std) (linalg.py:76-152): SplitMix64 uniforms in
    (0, 1] (53-bit), Box-Muller on the first / second half of the stream — the same bytes as the reference,
    so adapters attached here start from the factors the reference's attach_adapters would draw."""
    total = rows * cols
    pairs = (total + 1) // 2
    steps = np.arange(1, 2 * pairs + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + steps * np.uint64(_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        z = z ^ (z >> np.uint64(31))
    u = ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
    rad = np.sqrt(-2.0 * np.log(u[:pairs]))
    ang = 2.0 * np.pi * u[pairs:]
    flat = np.empty(2 * pairs)
    flat[0::2] = rad * np.cos(ang)
    flat[1::2] = rad * np.sin(ang)
    return (flat[:total] * std).reshape(rows, cols).astype(dtype)


# --------------------------------------------------------------------------- the numpy <-> device shim
_ZERO_BASES: dict = {}


def _zero_base(rows: int, cols: int, bits: int, device) -> QuantizedMatrix:
    """A quantised grid whose dequantised value is exactly 0 (codes, scale, offset all zero): the device
    adapter over it yields the adapter term alone (y2 = x·W_tᵀ, dx = dy·W_t) through the same kernels."""
    key = (rows, cols, bits, str(device))
    q = _ZERO_BASES.get(key)
    if q is None:
        ld = cols if bits == 8 else (cols + 1) // 2
        z = torch.zeros
        q = QuantizedMatrix(rows, cols, bits, z((rows, ld), dtype=torch.uint8, device=device),
                            z(rows, dtype=torch.float32, device=device), z(rows, dtype=torch.float32, device=device),
                            z(rows, dtype=torch.int32, device=device))
        _ZERO_BASES[key] = q
    return q


class HostLinear:
    """A device backend (QuantizedLinear / TTLinear / LoraLinear) behind the reference's numpy protocol:
    `kind`, `name`, `fan_in`, `fan_out`, `params()`, `forward(x, step)`, `backward(x, dy, grads, step)`,
    `astype`, `merged`.  The host Params (numpy) are the source of truth for the adapter factors — the
    reference's optimizer updates them in place — and are uploaded before every call (they are small);
    gradients come back as numpy arrays accumulated like _accumulate (transformer.py:150-156)."""

    def __init__(self, backend, act_quant: bool = True):
        self.backend = backend
        self.act_quant = bool(act_quant)
        self.name = backend.name
        self.kind = backend.kind
        self._host = []
        for p in backend.params():
            self._host.append(Param(p.name, p.data.detach().cpu().numpy().copy(), p.trainable))

    @property
    def fan_in(self):
        return self.backend.fan_in

    @property
    def fan_out(self):
        return self.backend.fan_out

    @property
    def merged(self):
        return getattr(self.backend, "merged", False)

    @property
    def q(self) -> QuantizedMatrix:
        b = self.backend
        return b.q if isinstance(b, QuantizedLinear) else b.base.q

    def params(self):
        return list(self._host)

    def astype(self, dtype):
        # like QuantizedLinear.astype (transformer.py:272-273): the device backend keeps its precision
        return self

    def _sync(self):
        """Upload the host factors into the device backend's tensors."""
        for hp, dp in zip(self._host, self.backend.params()):
            dp.data.copy_(torch.from_numpy(np.ascontiguousarray(hp.data, dtype=np.float32)))
            dp.trainable = hp.trainable

    def _adapter(self):
        b = self.backend
        return None if isinstance(b, QuantizedLinear) else (b.spec, b._core_tensors())

    @staticmethod
    def _dev(a) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.float32)).cuda()

    def forward(self, x, step: int = 0):
        x = np.asarray(x)
        xd = self._dev(x)
        self._sync()
        b = self.backend
        if getattr(b, "merged", False):
            y = b.forward(xd, step)
        elif self.act_quant:
            y = linear_forward(self.q, self._adapter(), xd)
        else:
            y = qmatmul(self.q, xd)
            ad = self._adapter()
            if ad is not None:
                y = y + linear_forward(_zero_base(self.q.rows, self.q.cols, self.q.bits, xd.device), ad, xd)
        return y.float().cpu().numpy().astype(x.dtype if x.dtype.kind == "f" else np.float32, copy=False)

    def backward(self, x, dy, grads, step: int = 0):
        dy = np.asarray(dy)
        dyd = self._dev(dy)
        self._sync()
        b = self.backend
        if getattr(b, "merged", False):
            raise ModelError(f"{self.name}: merged adapter is inference-only")
        ad = self._adapter()
        if ad is None:
            dx = linear_backward(self.q, None, None, dyd)[0] if self.act_quant else qmatmul_t(self.q, dyd)
        else:
            xd = self._dev(x)
            if self.act_quant:
                dx, dcores = linear_backward(self.q, ad, xd, dyd)
            else:
                zq = _zero_base(self.q.rows, self.q.cols, self.q.bits, dyd.device)
                dxa, dcores = linear_backward(zq, ad, xd, dyd)
                dx = qmatmul_t(self.q, dyd) + dxa
            self._scatter(grads, dcores)
        return dx.float().cpu().numpy().astype(dy.dtype if dy.dtype.kind == "f" else np.float32, copy=False)

    def _scatter(self, grads: dict, dcores):
        b = self.backend
        if isinstance(b, LoraLinear):
            r, k = b.down.data.shape
            n = b.up.data.shape[0]
            gs = [dcores[0].reshape(k, r).t(), dcores[1].reshape(r, n).t()]
        else:
            gs = list(dcores)
        for hp, g in zip(self._host, gs):
            _accumulate(grads, hp, g.contiguous().cpu().numpy())


def _unwrap(mat):
    return mat.backend if isinstance(mat, HostLinear) else mat


def _device_quantized(mat, device="cuda") -> QuantizedLinear:
    """A reference QuantizedLinear (numpy QuantizedMatrix) or a device one -> device QuantizedLinear, codes byte
    for byte (no re-quantisation)."""
    from .checkpoint import quantized_from_arrays

    m = _unwrap(mat)
    if isinstance(m, QuantizedLinear):
        return m
    q = getattr(m, "q", None)
    if q is None or getattr(m, "kind", None) != "quantized":
        raise ModelError(f"{getattr(m, 'name', m)}: not a quantized linear")
    return QuantizedLinear(m.name, quantized_from_arrays(q.codes, q.scale, q.offset, q.rows, q.cols, q.bits, device))


def _rebuild(model, convert):
    """A model of the caller's classes with every slot passed through convert(slot_name, mat)."""
    layer_cls = type(model.layers[0]) if model.layers else None
    layers = [layer_cls(layer.index, layer.norm1, layer.norm2,
                        {k: convert(k, m) for k, m in layer.matrices().items()}) for layer in model.layers]
    head = convert("wh", model.head)
    return type(model)(model.config, dict(model.specs), model.embed, layers, head, model.dtype)


def _check_targets(targets, we_error: str):
    targets = tuple(targets)
    for t in targets:
        if t == "we":
            raise ModelError(we_error)
        if t not in MATRIX_NAMES:
            raise ModelError(f"unknown matrix name {t!r}")
    return targets


def _set_spec(specs: dict, name: str, model, **kw):
    """LayerSpec of the caller's package (the class of an existing spec), if the model carries specs."""
    proto = next(iter(specs.values()), None)
    if proto is not None:
        specs[name] = type(proto)(**kw)


def to_device(model, act_quant: bool = True):
    """Every quantised slot of a reference model (QuantizedLinear, LoraLinear over a QuantizedLinear base) as a
    HostLinear over the device backend (codes byte for byte, factors copied); dense slots stay on the host."""

    def convert(name, mat):
        m = _unwrap(mat)
        if isinstance(m, (QuantizedLinear, TTLinear)):
            return mat if isinstance(mat, HostLinear) and mat.act_quant == act_quant else HostLinear(m, act_quant)
        if getattr(m, "kind", None) == "quantized":
            return HostLinear(_device_quantized(m), act_quant)
        if getattr(m, "kind", None) == "lora" and getattr(getattr(m, "base", None), "kind", None) == "quantized":
            base = _device_quantized(m.base)
            lora = LoraLinear(m.name, QuantizedLinear(m.base.name, base.q), np.asarray(m.down.data, np.float32),
                              np.asarray(m.up.data, np.float32))
            lora.down.trainable, lora.up.trainable = m.down.trainable, m.up.trainable
            return HostLinear(lora, act_quant)
        return mat

    return _rebuild(model, convert)


def quantize_model(model, bits: int, targets=None, act_quant: bool = True):
    """quantize_model (transformer.py:1114-1139) onto the device: targeted dense slots (`weight.data`) become
    device QuantizedLinear backends (qa_quantize_rows, bit-exact with quantize_rows) behind HostLinear."""
    targets = _check_targets(targets or ("wq", "wk", "wv", "wo", "wu", "wg", "wd", "wh"), "quantized embedding lookup is not supported")
    specs = dict(model.specs)

    def convert(name, mat):
        if name not in targets:
            return mat
        if getattr(mat, "kind", None) != "dense":
            raise ModelError(f"{mat.name}: only dense matrices can be quantized, found {mat.kind}")
        w = torch.from_numpy(np.ascontiguousarray(mat.weight.data, dtype=np.float32)).cuda()
        return HostLinear(QuantizedLinear(mat.name, quantize_rows(w, bits)), act_quant)

    out = _rebuild(model, convert)
    for name in targets:
        _set_spec(specs, name, model, kind="quantized", bits=bits)
    out.specs = specs
    return out


def attach_adapters(model, r: int, targets=("wq", "wv"), seed: int = 0, kind: str = "lora", spec_for=None,
                    act_quant: bool = True):
    """attach_adapters (lowrank.py:189-234) with device adapters over quantised bases.

    kind="lora": down ~ seeded N(0, 0.02²) drawn exactly as the reference draws it (seed * 7919 + counter),
    up = 0 (the identity delta).  kind="tt": the paper's tensor-train adapter with the pinned modes
    (TTSpec.for_shape, or spec_for(fan_out, fan_in, r)); cores ~ seeded N(0, 0.02²) with the last core zero.
    Rejects the embedding, unknown names, rank >= min(fan_in, fan_out) and non-quantised bases (the device
    adapters run on the int8 / int4 codes)."""
    targets = _check_targets(targets, "adapters on the embedding lookup are not supported")
    if kind not in ("lora", "tt"):
        raise ModelError(f"unknown adapter kind {kind!r}")
    counter = [0]
    specs = dict(model.specs)

    def wrap(name, mat):
        if name not in targets:
            return mat
        counter[0] += 1
        m = _unwrap(mat)
        if getattr(m, "kind", None) != "quantized":
            raise ModelError(f"{getattr(m, 'name', name)}: device adapters need a quantized base, found "
                             f"{getattr(m, 'kind', type(m).__name__)} (quantize_model first)")
        base = QuantizedLinear(m.name + ".base", _device_quantized(m).q)
        fan_out, fan_in = base.fan_out, base.fan_in
        if r >= min(fan_in, fan_out):
            raise ModelError(f"{m.name}: rank {r} must be < min(fan_in, fan_out)")
        if kind == "lora":
            down = seeded_gaussian(r, fan_in, seed * 7919 + counter[0], std=INIT_STD)
            up = np.zeros((fan_out, r), dtype=np.float32)
            return HostLinear(LoraLinear(m.name, base, down, up), act_quant)
        spec = spec_for(fan_out, fan_in, r) if spec_for is not None else TTSpec.for_shape(fan_out, fan_in, r)
        cores = []
        for k in range(spec.d):
            shp = spec.core_shape(k)
            c = seeded_gaussian(int(np.prod(shp[:2])), int(np.prod(shp[2:])), (seed * 7919 + counter[0]) * 8 + k,
                                std=INIT_STD).reshape(shp)
            cores.append(torch.from_numpy(np.zeros_like(c) if k == spec.d - 1 else c).cuda())
        return HostLinear(TTLinear(m.name, base, spec, cores), act_quant)

    out = _rebuild(model, wrap)
    for t in targets:
        _set_spec(specs, t, model, kind="lora", r=r)
    out.specs = specs
    return out


def configure_trainable(model, method: str = "lora_finetune"):
    """configure_trainable (trainer.py:124-151) for models with device adapters: "lora_finetune" trains only
    the adapter factors (LoRA down / up, tensor-train cores), every other tensor is frozen; other methods
    train everything that is not a frozen base."""
    adapters = set()
    mats = [m for layer in model.layers for m in layer.matrices().values()] + [model.head]
    for mat in mats:
        m = _unwrap(mat)
        if isinstance(m, TTLinear) or getattr(m, "kind", None) == "lora":
            adapters.update(p.name for p in mat.params() if not p.name.endswith(".weight"))
    if method == "lora_finetune" and not adapters:
        raise ModelError("lora_finetune requires adapters on at least one matrix")
    for p in model.named_parameters().values():
        p.trainable = (p.name in adapters) if method == "lora_finetune" else not p.name.endswith(".base")
    return model


def merge_model(model):
    """merge_model (lowrank.py:260-281) through the explicit dequantise route lowrank.py:249-252 prescribes:
    every device adapter folds into W' = deq(codes) + W_t (tt_merge, fp32) and serves the dense bf16 forward;
    a second merge raises, and a merged slot's backward raises (inference-only), as in the reference."""
    specs = dict(model.specs)

    def fold(name, mat):
        m = _unwrap(mat)
        if isinstance(m, TTLinear):
            if isinstance(mat, HostLinear):
                mat._sync()
            tt_merge(m)
            _set_spec(specs, name, model, kind="dense")
            return mat if isinstance(mat, HostLinear) else HostLinear(m)
        return mat

    out = _rebuild(model, fold)
    out.specs = specs
    return out
