"""Decoder stack with per-layer recompute (BASELINE config 4) against a CPU float64 restatement
of the reference's model_forward / model_backward (transformer.py:858-1007): torch float64 autograd for the
glue (RMSNorm :478-497, RoPE :499-519, causal softmax attention, SiLU gating, residuals, mean cross-entropy
:569-588) and the oracle's qa_linear_forward / qa_linear_backward for every linear (embedding table, weights
and adapter cores copied from the device model).

The float64 run rounds to bf16 wherever the device path stores a bf16 activation (norm outputs, linear
outputs, rotated q/k, attention context, gated activation, residual stream) — forward values and, through
the cast's autograd, the gradients at the same points — so both runs quantise nearly the same activations.
What remains is bf16 arithmetic inside kernels (linear dx, the attention kernel's bf16 P / dS tiles) and the
act-quant code flips it causes, compounded over the layers.  Measured on this 2-layer case: the reference
with vs without the bf16 emulation differs by up to 0.044 (norm-relative) per gradient tensor — the noise
floor of bf16 activation storage — and the device path sits below it (0.037 with the cuDNN attention,
0.013 with a float32 attention).  Bars (per adapter-gradient tensor, ||got - want|| / ||want||):
  NORM_TOL 5e-2 with the library attention, NORM_TOL_F32ATT 2e-2 with float32 attention (isolates this
  package's kernels); loss within 1e-4 relative.
PER_LAYER and STORE_ALL on the device agree to 1e-3 (attention backward may accumulate in any order).
"""

import numpy as np
import pytest
import torch

import oracle as O
from paper_2402_13533_b200 import decoder
from paper_2402_13533_b200.decoder import DecoderConfig, build_decoder

pytestmark = pytest.mark.gpu

NORM_TOL = 5e-2
NORM_TOL_F32ATT = 2e-2
CFG = DecoderConfig(vocab=512, dim=256, heads=2, layers=2, ffn_dim=512, max_seq=64)


def _oquant(q):
    h = q.to_numpy()
    return O.OQuant(rows=q.rows, cols=q.cols, bits=q.bits, codes=h["codes"], scale=h["scale"], offset=h["offset"])


class _OracleLinear(torch.autograd.Function):
    """One reference linear (TT adapter over a quantised base) on the oracle, float64."""

    @staticmethod
    def forward(ctx, x, oq, cores, grads, name):
        ctx.oq, ctx.cores, ctx.grads, ctx.name = oq, cores, grads, name
        ctx.save_for_backward(x)
        lead = x.shape[:-1]
        y = O.qa_linear_forward(x.numpy(), oq, cores)["y"]
        return torch.from_numpy(y).reshape(*lead, oq.rows)

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        r = O.qa_linear_backward(x.numpy(), dy.contiguous().numpy(), ctx.oq, ctx.cores)
        for k, g in enumerate(r["dcores"]):
            key = f"{ctx.name}.core{k}"
            ctx.grads[key] = ctx.grads.get(key, 0) + g
        return torch.from_numpy(r["dx"]).reshape(x.shape), None, None, None, None


def _reference(model, tokens, targets):
    cfg = model.config
    grads = {}
    lin = {}
    for li, layer in enumerate(model.layers):
        for k, m in layer.mats.items():
            lin[m.name] = (_oquant(m.base.q), [c.data.double().cpu().numpy() for c in m.cores])
    lin["head"] = (_oquant(model.head.base.q), [c.data.double().cpu().numpy() for c in model.head.cores])

    def R(t):  # the device path's bf16 activation storage
        return t.to(torch.bfloat16).to(torch.float64)

    def linear(name, x):
        oq, cores = lin[name]
        return R(_OracleLinear.apply(x, oq, cores, grads, name))

    b, l = tokens.shape
    d = cfg.head_dim
    half = d // 2
    freqs = cfg.rope_base ** (-2.0 * torch.arange(half, dtype=torch.float64) / d)
    ang = torch.arange(l, dtype=torch.float64)[:, None] * freqs[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def rms(x):
        return x / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-5)

    def rope(x):
        xh = x.reshape(b, l, cfg.heads, half, 2)
        e, o = xh[..., 0], xh[..., 1]
        c, s = cos[None, :, None, :], sin[None, :, None, :]
        return torch.stack((e * c - o * s, e * s + o * c), -1).reshape(b, l, cfg.dim)

    def heads(t):
        return t.reshape(b, l, cfg.heads, d).transpose(1, 2)

    mask = torch.triu(torch.full((l, l), float("-inf"), dtype=torch.float64), 1)
    x = model.embed[tokens.cuda()].double().cpu().requires_grad_(True)
    for li, layer in enumerate(model.layers):
        p = f"layers.{li}."
        n1 = R(rms(x))
        q, k, v = (linear(p + nm, n1) for nm in ("wq", "wk", "wv"))
        q, k = R(rope(q)), R(rope(k))
        s = torch.softmax(heads(q) @ heads(k).transpose(-1, -2) / np.sqrt(d) + mask, -1)
        ctx = R((s @ heads(v)).transpose(1, 2).reshape(b, l, cfg.dim))
        res1 = R(x + linear(p + "wo", ctx))
        n2 = R(rms(res1))
        act = R(linear(p + "wu", n2) * torch.nn.functional.silu(linear(p + "wg", n2)))
        x = R(res1 + linear(p + "wd", act))
    logits = linear("head", x).reshape(b * l, cfg.vocab)
    loss = torch.nn.functional.cross_entropy(logits, targets.reshape(-1).cpu())
    loss.backward()
    return float(loss.detach()), grads


@pytest.fixture(scope="module")
def setup():
    model = build_decoder(CFG, rank=8, bits=8, seed=3)
    g = torch.Generator().manual_seed(11)
    tokens = torch.randint(0, CFG.vocab, (2, CFG.max_seq), generator=g).cuda()
    targets = torch.randint(0, CFG.vocab, (2, CFG.max_seq), generator=g).cuda()
    return model, tokens, targets


def _norm_rel(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))


def _f32_attention(q, k, v, is_causal=True):
    l = q.shape[-2]
    s = (q.float() @ k.float().transpose(-1, -2)) / (q.shape[-1] ** 0.5)
    s = s + torch.triu(torch.full((l, l), float("-inf"), device=q.device), 1)
    return (torch.softmax(s, -1) @ v.float()).to(q.dtype)


@pytest.mark.parametrize("attention", ["library", "float32"])
def test_decoder_per_layer_matches_reference(setup, attention, monkeypatch):
    model, tokens, targets = setup
    if attention == "float32":
        monkeypatch.setattr(decoder.F, "scaled_dot_product_attention", _f32_attention)
    loss, grads = model.train_step_grads(tokens, targets)
    want_loss, want = _reference(model, tokens.cpu(), targets)
    assert abs(loss - want_loss) <= 1e-4 * abs(want_loss)
    names = {p.name for m in model.adapters() for p in m.cores}
    assert set(grads) == names == set(want)
    tol = NORM_TOL if attention == "library" else NORM_TOL_F32ATT
    errs = {k: _norm_rel(grads[k].cpu().numpy(), want[k]) for k in sorted(names)}
    bad = {k: e for k, e in errs.items() if not e < tol}
    assert not bad, (bad, max(errs.values()))


def test_decoder_per_layer_equals_store_all(setup):
    model, tokens, targets = setup
    l1, g1 = model.train_step_grads(tokens, targets, policy="per_layer")
    l2, g2 = model.train_step_grads(tokens, targets, policy="store_all")
    assert l1 == pytest.approx(l2, rel=1e-6)
    assert set(g1) == set(g2)
    for k in g1:
        assert O.rel_err(g1[k].cpu().numpy(), g2[k].cpu().numpy()) < 1e-3, k


def test_decoder_rejects_long_sequences(setup):
    model, tokens, targets = setup
    long = torch.zeros((1, CFG.max_seq + 1), dtype=torch.long, device="cuda")
    with pytest.raises(ValueError):
        model.train_step_grads(long, long)


def test_decoder_train_step_updates_adapters_only(setup):
    """train_step = grads + AdamW (trainer.py:165-199): the kernels accumulate the core gradients straight into
    the optimizer's flat buffer (equal to the dict path's gradients up to the attention kernel's accumulation
    order), every adapter core moves, and the embedding / quantised bases do not."""
    from paper_2402_13533_b200.optim import AdamWConfig

    model, tokens, targets = setup
    params = model.trainable()
    before = {k: p.data.clone() for k, p in params.items()}
    embed0 = model.embed.clone()
    codes0 = model.layers[0].mats["wq"].base.q.codes.clone()
    _, want = model.train_step_grads(tokens, targets)
    loss, st = model.train_step(tokens, targets, config=AdamWConfig(lr=1e-3))
    assert st.step == 1 and loss > 0
    views = st._grad_views
    for k in params:
        assert O.rel_err(views[k].cpu().numpy(), want[k].cpu().numpy()) < 1e-3, k
        assert params[k].data.data_ptr() != before[k].data_ptr()
        assert not torch.equal(params[k].data, before[k]), k
    assert torch.equal(model.embed, embed0)
    assert torch.equal(model.layers[0].mats["wq"].base.q.codes, codes0)
    loss2, st2 = model.train_step(tokens, targets, st, config=AdamWConfig(lr=1e-3))
    assert st2 is st and st.step == 2 and loss2 < loss


def test_decoder_matches_reference_model_backward():
    """Drop-in proof against the REFERENCE itself: tests/golden/decoder_small.npz holds a
    2-layer lrlm model (quantize_model(8) on every linear and the head, attach_adapters LoRA r = 8 on all of
    them, lora_finetune) and the loss and gradient dict of its own model_forward(PER_LAYER) /
    model_backward (oracle/gen_decoder_golden.py).  The same bases (codes byte for byte), factors, embedding
    and tokens run through DecoderStack with the device LoraLinear backends: the gradient dict has the
    reference's keys and every tensor agrees to 5e-2 (norm-relative).  The gap is the paper's per-token
    activation quantisation, which the reference's QuantizedLinear does not apply (qmatmul on float x,
    quant.py:123-132), plus bf16 activation storage; the loss agrees to 1e-2."""
    import os

    from paper_2402_13533_b200.checkpoint import quantized_from_arrays
    from paper_2402_13533_b200.decoder import DecoderLayer, DecoderStack
    from paper_2402_13533_b200.linear import LoraLinear, QuantizedLinear

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "decoder_small.npz"))
    vocab, dim, heads, layers, ffn, max_seq = (int(v) for v in g["config"])
    cfg = DecoderConfig(vocab=vocab, dim=dim, heads=heads, layers=layers, ffn_dim=ffn, max_seq=max_seq)

    def lora(path):
        down, up = g[f"{path}.down"], g[f"{path}.up"]
        rows, cols = up.shape[0], down.shape[1]
        q = quantized_from_arrays(g[f"{path}.codes"], g[f"{path}.scale"], g[f"{path}.offset"], rows, cols, 8)
        return LoraLinear(path, QuantizedLinear(path + ".base", q), torch.from_numpy(down), torch.from_numpy(up))

    ones = torch.ones(dim, device="cuda")
    stack = [DecoderLayer(i, ones, ones, {k: lora(f"layers.{i}.{k}") for k in ("wq", "wk", "wv", "wo", "wu", "wg",
                                                                             "wd")})
             for i in range(layers)]
    model = DecoderStack(cfg, torch.from_numpy(g["embed"]).cuda().to(torch.bfloat16), stack, lora("head"))
    tokens = torch.from_numpy(g["tokens"]).cuda()
    targets = torch.from_numpy(g["targets"]).cuda()
    loss, grads = model.train_step_grads(tokens, targets)
    want = {k[len("grad::"):]: g[k] for k in g.files if k.startswith("grad::")}
    assert sorted(grads) == sorted(want)
    assert abs(loss - float(g["loss"])) <= 1e-2 * abs(float(g["loss"]))
    errs = {k: _norm_rel(grads[k].cpu().numpy(), want[k]) for k in want}
    bad = {k: e for k, e in errs.items() if not e < 5e-2}
    assert not bad, (bad, max(errs.values()))


def _f32_sdpa(q, k, v, is_causal=False):
    s = (q.float() @ k.float().transpose(-1, -2)) / (q.shape[-1] ** 0.5)
    if is_causal:
        lq, lk = q.shape[-2], k.shape[-2]
        s = s + torch.triu(torch.full((lq, lk), float("-inf"), device=q.device), 1)
    return (torch.softmax(s, -1) @ v.float()).to(q.dtype)


def test_kv_decode_matches_full_forward_and_greedy(setup, monkeypatch):
    """kv_decode_step (transformer.py:1043-1080) on the device: the logits of each cached one-token step equal the
    matching position of a full forward over the prefix (the reference's own contract for the cache).  Both paths
    run the same float32 attention here.  For a prefix of <= 8 tokens the full forward's linears take the same
    decode-size kernels (act-quant prologue + matrix-vector pass) as the one-token steps: bit-identical logits at
    every position.  Longer prefixes run the tcgen05 path, whose adapter term (3-term bf16 split GEMM) differs
    from the prologue's fp32 chain in the last bits; rare bf16 / act-quant code flips then compound over the layers
    (measured up to 4e-2 max-normalised on this random model after the train-step test moved the cores).
    greedy_decode with and without the cache agree."""
    model, tokens, _ = setup
    monkeypatch.setattr(decoder.F, "scaled_dot_product_attention", _f32_sdpa)
    for n, bar in ((8, 0.0), (12, 0.1)):
        seq = tokens[0, :n].tolist()
        full = model.forward(torch.tensor([seq], device="cuda"))[0].float()
        cache = decoder.KvCache(model)
        errs = []
        for i, t in enumerate(seq):
            logits, cache = decoder.kv_decode_step(model, cache, t)
            assert logits.shape == (CFG.vocab,) and logits.dtype == torch.float32
            errs.append(O.rel_err(logits.cpu().numpy(), full[i].cpu().numpy()))
        print(f"kv decode vs full forward ({n} tokens):", " ".join(f"{e:.1e}" for e in errs))
        assert max(errs) <= bar, errs
        assert cache.current_len == n
    with pytest.raises(decoder.ModelError, match="out of range"):
        decoder.kv_decode_step(model, cache, CFG.vocab)
    gen, passes = decoder.greedy_decode(model, seq[:4], max_new=5)
    gen2, passes2 = decoder.greedy_decode(model, seq[:4], max_new=5, use_cache=False)
    assert passes == 4 + 4 and passes2 == sum(4 + i for i in range(5))
    assert gen == gen2
    over = decoder.KvCache(model)
    over.length = CFG.max_seq
    with pytest.raises(decoder.ModelError, match="overflow"):
        decoder.kv_decode_step(model, over, 1)
