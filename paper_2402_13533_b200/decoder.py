"""Decoder-layer stack over the quantised tensor-adapter linears with per-layer recompute (SURVEY §8(f) 2,
BASELINE config 4): `_layer_forward` / `_layer_backward` / `model_forward` / `model_backward` of the reference
(transformer.py:858-1007) on the device.

Every step is this package's kernels except causal attention, which is torch's scaled-dot-product attention
(a library kernel, differentiated by autograd inside the layer's recompute window):
  - the linears: q/k/v on norm1 and up/gate on norm2 as shared-input groups (one act-quant / Z1 pass over
    the input per direction), each recompute-forward handing Z1 to its backward;
  - the glue (glue.py / csrc/glue.cu): rmsnorm with the residual add folded in, its backward with the group's
    summed dx and the residual gradient folded in, in-place RoPE, SiLU gating, fused cross-entropy.
The PER_LAYER policy (:613-637) keeps each layer's input and the final hidden state; the backward re-runs one
layer's forward (keeping its activations) right before that layer's backward.  STORE_ALL keeps every layer's
activations (tests compare the two, like the reference's recompute tests).
Only adapter cores are trainable (configure_trainable("lora_finetune"), trainer.py:133-147); norm gains and the
embedding are frozen; gradients accumulate in a dict keyed by the cores' names, like _accumulate.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import dp, glue
from .optim import AdamWConfig, AdamWState, adamw_step
from .linear import ModelError, QuantizedLinear, TTLinear, TTSpec, attach_tt_adapter, group_backward, group_forward
from .quant import quantize_rows

__all__ = ["DecoderConfig", "DecoderLayer", "DecoderStack", "KvCache", "build_decoder", "kv_decode_step",
           "greedy_decode"]


@dataclass(frozen=True)
class DecoderConfig:
    """The reference's ModelConfig fields (transformer.py:65-101)."""

    vocab: int
    dim: int
    heads: int
    layers: int
    ffn_dim: int
    max_seq: int
    rope_base: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads


def _group_fwd(members, x):
    return group_forward(members, x) if len(members) > 1 else [members[0].forward(x)]


def _group_bwd(members, x, dys, grads):
    if len(members) > 1:
        return group_backward(members, x, dys, grads)
    return [members[0].backward(x, dys[0], grads)]


class DecoderLayer:
    """One pre-norm decoder layer (transformer.py:660-690): norm1 -> q/k/v (RoPE on q, k) -> causal attention
    -> wo -> residual -> norm2 -> up/gate -> SiLU gating -> wd -> residual."""

    def __init__(self, index, norm1, norm2, mats: dict):
        self.index = index
        self.norm1, self.norm2 = norm1, norm2  # frozen f32 gains
        self.mats = mats  # wq wk wv wo wu wg wd -> TTLinear

    def forward(self, x, shape, rope, keep: bool):
        """_layer_forward (transformer.py:858-880).  x: [T, D] bf16 (T = batch * seq).  Returns (out, entry);
        entry holds what _layer_backward reads when keep is True (else None)."""
        b, l, heads = shape
        T, D = x.shape
        d = D // heads
        m = self.mats
        norm1, inv1 = glue.rmsnorm(x, self.norm1)
        q, k, v = _group_fwd([m["wq"], m["wk"], m["wv"]], norm1)
        glue.rope_(q, k, rope[0], rope[1], heads, l)

        def split(t):
            return t.view(b, l, heads, d).transpose(1, 2)

        if keep:
            q.requires_grad_(True)
            k.requires_grad_(True)
            v.requires_grad_(True)
            with torch.enable_grad():
                ctx_g = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
                ctx_g = ctx_g.transpose(1, 2).reshape(T, D)
            ctx = ctx_g.detach()
        else:
            ctx_g = None
            ctx = F.scaled_dot_product_attention(split(q), split(k), split(v), is_causal=True)
            ctx = ctx.transpose(1, 2).reshape(T, D)
        if not ctx.is_contiguous():
            ctx = ctx.contiguous()
        (attn,) = _group_fwd([m["wo"]], ctx)
        norm2, inv2, res1 = glue.rmsnorm(x, self.norm2, b=attn)
        up, gate = _group_fwd([m["wu"], m["wg"]], norm2)
        act = glue.swiglu(up, gate)
        (ffn,) = _group_fwd([m["wd"]], act)
        out = res1 + ffn
        if not keep:
            return out, None
        return out, {"x": x, "norm1": norm1, "inv1": inv1, "q": q, "k": k, "v": v, "ctx_g": ctx_g, "ctx": ctx,
                     "res1": res1, "norm2": norm2, "inv2": inv2, "up": up, "gate": gate, "act": act}

    def backward(self, e, dout, shape, rope, grads):
        """_layer_backward (transformer.py:910-946): returns dx, accumulates the adapter-core gradients."""
        b, l, heads = shape
        m = self.mats
        (dact,) = _group_bwd([m["wd"]], e["act"], [dout], grads)
        dup, dgate = glue.swiglu_backward(e["up"], e["gate"], dact)
        dn2 = _group_bwd([m["wu"], m["wg"]], e["norm2"], [dup, dgate], grads)
        dres1 = glue.rmsnorm_backward(e["res1"], self.norm2, e["inv2"], dn2, dres=dout)
        (dctx,) = _group_bwd([m["wo"]], e["ctx"], [dres1], grads)
        dq, dk, dv = torch.autograd.grad(e["ctx_g"], (e["q"], e["k"], e["v"]), dctx)
        dq, dk, dv = dq.contiguous(), dk.contiguous(), dv.contiguous()
        glue.rope_(dq, dk, rope[0], rope[1], heads, l, inverse=True)
        dn1 = _group_bwd([m["wq"], m["wk"], m["wv"]], e["norm1"], [dq, dk, dv], grads)
        return glue.rmsnorm_backward(e["x"], self.norm1, e["inv1"], dn1, dres=dres1)


class DecoderStack:
    """embed -> layers -> quantised head with adapter (transformer.py:949-1007); no final norm, like the
    reference's model_forward."""

    def __init__(self, config: DecoderConfig, embed, layers, head: TTLinear):
        self.config, self.embed, self.layers, self.head = config, embed, layers, head

    def adapters(self):
        out = [m for layer in self.layers for m in layer.mats.values()]
        return out + [self.head]

    def trainable(self) -> dict:
        """name -> Param of every adapter core (configure_trainable("lora_finetune"), trainer.py:133-147)."""
        return {p.name: p for m in self.adapters() for p in m.params() if p.trainable}

    def train_step(self, tokens, targets, state: AdamWState | None = None, config: AdamWConfig | None = None,
                   micro_batches: int = 1, process_group=None):
        """trainer.train_step (trainer.py:165-199) with the PER_LAYER policy: per micro-batch (np.array_split
        of the rows) forward, cross-entropy and backward with recompute, gradients summed and divided by the
        micro-batch count, then one AdamW update of the adapter cores.  With a torch.distributed process
        group of G > 1 ranks (data parallelism, each rank holding its shard of the batch), the flat gradient
        buffer is all-reduced and divided by G before the update (the fixed-order average of
        distsim.federated_round, distsim.py:309-314), so every replica applies the same update.
        Returns (mean loss of this rank's shard, state)."""
        params = self.trainable()
        if state is None:
            state = AdamWState(params)
        if micro_batches < 1:
            raise ValueError("micro_batches must be >= 1")
        # cores live in the optimizer's flat float32 buffer and the kernels accumulate their gradients
        # straight into its flat gradient buffer (no per-tensor gather / copy-back around the update)
        if getattr(state, "_bound_to", None) is not self:
            if process_group is not None:  # replicas must start identical (distsim.py:293-296)
                dp.check_replicas(self.adapters(), process_group)
            state._grad_views = state.bind(params)
            state._bound_to = self
        state.gflat.zero_()
        total = dict(state._grad_views)
        loss_sum = 0.0
        b = tokens.shape[0]
        sizes = [b // micro_batches + (1 if i < b % micro_batches else 0) for i in range(micro_batches)]
        start = 0
        for n in sizes:
            loss, _ = self.train_step_grads(tokens[start:start + n], targets[start:start + n], grads=total)
            start += n
            loss_sum += loss
        dp.average_flat_(state.gflat, micro_batches, process_group)
        adamw_step(state, params, total, config or AdamWConfig())
        return loss_sum / micro_batches, state

    def rope_tables(self, length, device):
        """_rope_tables (transformer.py:499-503): angles in float64, tables stored as float32."""
        d = self.config.head_dim
        half = d // 2
        freqs = self.config.rope_base ** (-2.0 * torch.arange(half, dtype=torch.float64, device=device) / d)
        ang = torch.arange(length, dtype=torch.float64, device=device)[:, None] * freqs[None, :]
        return torch.cos(ang).float().contiguous(), torch.sin(ang).float().contiguous()

    def forward(self, tokens):
        """model_forward (transformer.py:949-981) for inference: logits [batch, seq, vocab] (bf16), no tape."""
        cfg = self.config
        tokens = torch.as_tensor(tokens, device=self.embed.device)
        if tokens.dim() == 1:
            tokens = tokens[None]
        b, l = tokens.shape
        if l > cfg.max_seq:
            raise ModelError(f"sequence length {l} exceeds max_seq {cfg.max_seq}")
        if int(tokens.min()) < 0 or int(tokens.max()) >= cfg.vocab:
            raise ModelError(f"token id out of range [0, {cfg.vocab})")
        shape = (b, l, cfg.heads)
        rope = self.rope_tables(l, tokens.device)
        x = self.embed[tokens.reshape(-1)]
        for layer in self.layers:
            x, _ = layer.forward(x, shape, rope, keep=False)
        (logits,) = _group_fwd([self.head], x)
        return logits.view(b, l, -1)

    def train_step_grads(self, tokens, targets, policy: str = "per_layer", grads: dict | None = None):
        """One forward + cross-entropy + backward (model_forward / cross_entropy_grad / model_backward).
        policy "per_layer" keeps only each layer's input and recomputes; "store_all" keeps every layer's
        activations.  Gradients accumulate into `grads` (new dict if None; preallocated float32 tensors are
        accumulated into by the kernels).  Returns (loss, grads dict of the adapter cores)."""
        cfg = self.config
        if tokens.dim() != 2:
            raise ValueError(f"tokens must be 2-D, got shape {tuple(tokens.shape)}")
        b, l = tokens.shape
        if l > cfg.max_seq:
            raise ValueError(f"sequence length {l} exceeds max_seq {cfg.max_seq}")
        if policy not in ("per_layer", "store_all"):
            raise ValueError(f"unknown recompute policy {policy!r}")
        keep_all = policy == "store_all"
        shape = (b, l, cfg.heads)
        rope = self.rope_tables(l, tokens.device)
        grads = {} if grads is None else grads
        stored = []
        x = self.embed[tokens.reshape(-1)]
        for layer in self.layers:
            xin = x
            x, entry = layer.forward(x, shape, rope, keep=keep_all)
            stored.append(entry if keep_all else xin)
        (logits,) = _group_fwd([self.head], x)
        loss, dlogits = glue.cross_entropy(logits, targets)
        del logits
        (dx,) = _group_bwd([self.head], x, [dlogits], grads)
        del dlogits
        for layer, st in zip(reversed(self.layers), reversed(stored)):
            entry = st if keep_all else layer.forward(st, shape, rope, keep=True)[1]
            dx = layer.backward(entry, dx, shape, rope, grads)
            del entry
        return float(loss), grads


class KvCache:
    """Per-layer key / value grids in HBM, one row appended per decode step (transformer.py:1015-1027): bf16
    [max_seq, dim] per layer, as the projections produce them (k after RoPE)."""

    def __init__(self, model: "DecoderStack"):
        cfg = model.config
        dev = model.embed.device
        self.max_seq = cfg.max_seq
        self.length = 0
        self.k = [torch.zeros((cfg.max_seq, cfg.dim), dtype=torch.bfloat16, device=dev) for _ in range(cfg.layers)]
        self.v = [torch.zeros((cfg.max_seq, cfg.dim), dtype=torch.bfloat16, device=dev) for _ in range(cfg.layers)]
        self.rope = model.rope_tables(cfg.max_seq, dev)

    @property
    def current_len(self) -> int:
        return self.length


def kv_decode_step(model: "DecoderStack", cache: KvCache, token: int, step: int = 0):
    """kv_decode_step (transformer.py:1043-1080) on the device: exactly one token through the stack — each linear
    a decode-size forward (act-quant prologue + tensor-core matrix-vector pass; q/k/v and up/gate as shared-input
    groups), RoPE at this position, attention of the new query over the cached keys / values (torch SDPA), the
    cache grown by one row.  Returns (logits [vocab] f32, cache)."""
    cfg = model.config
    if cache.length >= cache.max_seq:
        raise ModelError(f"kv cache overflow: length {cache.length} at max_seq {cache.max_seq}")
    if not 0 <= int(token) < cfg.vocab:
        raise ModelError(f"token id {token} out of range")
    pos = cache.length
    heads, d = cfg.heads, cfg.head_dim
    cos, sin = cache.rope[0][pos:pos + 1], cache.rope[1][pos:pos + 1]
    x = model.embed[int(token)].reshape(1, cfg.dim).contiguous()
    for li, layer in enumerate(model.layers):
        m = layer.mats
        norm1, _ = glue.rmsnorm(x, layer.norm1)
        q, k, v = _group_fwd([m["wq"], m["wk"], m["wv"]], norm1)
        glue.rope_(q, k, cos, sin, heads, 1)
        cache.k[li][pos].copy_(k[0])
        cache.v[li][pos].copy_(v[0])
        keys = cache.k[li][:pos + 1].view(pos + 1, heads, d).transpose(0, 1)
        vals = cache.v[li][:pos + 1].view(pos + 1, heads, d).transpose(0, 1)
        ctx = F.scaled_dot_product_attention(q.view(heads, 1, d), keys, vals)
        ctx = ctx.reshape(1, cfg.dim).contiguous()
        (attn,) = _group_fwd([m["wo"]], ctx)
        norm2, _, res1 = glue.rmsnorm(x, layer.norm2, b=attn)
        up, gate = _group_fwd([m["wu"], m["wg"]], norm2)
        (ffn,) = _group_fwd([m["wd"]], glue.swiglu(up, gate))
        x = res1 + ffn
    cache.length += 1
    (logits,) = _group_fwd([model.head], x)
    return logits[0].float(), cache


def greedy_decode(model: "DecoderStack", prompt, max_new: int, use_cache: bool = True):
    """greedy_decode (transformer.py:1083-1111): greedy continuation of the prompt; returns (generated ids, token
    passes).  use_cache=False re-runs the full forward over the growing sequence for every new token."""
    prompt = [int(t) for t in torch.as_tensor(prompt).reshape(-1).tolist()]
    if not prompt:
        raise ModelError("prompt must hold at least one token")
    generated: list[int] = []
    passes = 0
    if use_cache:
        cache = KvCache(model)
        logits = None
        for tok in prompt:
            logits, cache = kv_decode_step(model, cache, tok)
            passes += 1
        for _ in range(max_new):
            nxt = int(torch.argmax(logits))
            generated.append(nxt)
            if len(generated) == max_new:
                break
            logits, cache = kv_decode_step(model, cache, nxt)
            passes += 1
    else:
        seq = list(prompt)
        dev = model.embed.device
        for _ in range(max_new):
            logits = model.forward(torch.tensor([seq], dtype=torch.int64, device=dev))
            passes += len(seq)
            nxt = int(torch.argmax(logits[0, -1]))
            generated.append(nxt)
            seq.append(nxt)
    return generated, passes


def build_decoder(cfg: DecoderConfig, rank: int = 8, bits: int = 8, seed: int = 0, device="cuda") -> DecoderStack:
    """Random-init decoder (weights ~N(0, 0.02), like build_model, transformer.py:805-855), every linear
    quantised (quantize_model, :1114-1133) with a TT adapter of the pinned modes (attach_adapters with
    targets = all seven linears + the head "wh", lowrank.py:189-234); bf16 embedding table, norm gains 1."""
    if cfg.dim % cfg.heads or cfg.head_dim % 8:
        raise ValueError("dim must split into heads of a multiple of 8 columns")
    g = torch.Generator(device=device).manual_seed(seed)
    embed = (torch.randn((cfg.vocab, cfg.dim), generator=g, device=device) * 0.02).to(torch.bfloat16)
    shapes = {"wq": (cfg.dim, cfg.dim), "wk": (cfg.dim, cfg.dim), "wv": (cfg.dim, cfg.dim), "wo": (cfg.dim, cfg.dim),
              "wu": (cfg.ffn_dim, cfg.dim), "wg": (cfg.ffn_dim, cfg.dim), "wd": (cfg.dim, cfg.ffn_dim)}
    layers = []
    for li in range(cfg.layers):
        mats = {}
        for name, (n, k) in shapes.items():
            w = torch.randn((n, k), generator=g, device=device) * 0.02
            base = QuantizedLinear(f"layers.{li}.{name}.base", quantize_rows(w, bits))
            del w
            mats[name] = attach_tt_adapter(f"layers.{li}.{name}", base, rank, seed=seed * 1000 + li * 10 + len(mats))
        ones = torch.ones(cfg.dim, device=device)
        layers.append(DecoderLayer(li, ones, ones, mats))
    w = torch.randn((cfg.vocab, cfg.dim), generator=g, device=device) * 0.02
    head_base = QuantizedLinear("head.base", quantize_rows(w, bits))
    del w
    head = attach_tt_adapter("head", head_base, rank, spec=TTSpec.for_shape(cfg.vocab, cfg.dim, rank), seed=seed + 7)
    return DecoderStack(cfg, embed, layers, head)
