"""Generate tests/golden/decoder_small.npz with the REFERENCE package (lrlm): one PER_LAYER training
forward / backward of a small quantised decoder with LoRA adapters on every linear and the head.

Test infrastructure only; run in the build container (it needs /root/reference):

    python oracle/gen_decoder_golden.py

The model is the reference's own: build_model (transformer.py:805-839) -> quantize_model(8) on all seven
linears and the head (:1114-1139) -> attach_adapters on all of them (lowrank.py:189-234, the zero `up`
factors replaced by seeded values so every factor gets a gradient) -> configure_trainable("lora_finetune")
(trainer.py:124-151); then model_forward(PER_LAYER) / cross_entropy_loss / cross_entropy_grad /
model_backward (transformer.py:569-588, :949-1007).  The npz holds every array the device model needs
(embedding table, u8 codes / scales / offsets of every base, LoRA factors), the tokens and targets, the
loss and the reference's gradient dict, so tests/test_gpu_decoder.py runs the same model through
paper_2402_13533_b200.decoder and compares (the drop-in proof of SURVEY §8(b)).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("LRLM_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
MATS = ("wq", "wk", "wv", "wo", "wu", "wg", "wd")


def main():
    sys.path.insert(0, REF)
    from lrlm import linalg, lowrank, trainer  # noqa: E402  (reference, read-only)
    from lrlm import transformer as tfm  # noqa: E402

    cfg = tfm.ModelConfig(vocab=512, dim=256, heads=2, layers=2, ffn_dim=512, max_seq=64)
    model = tfm.build_model(cfg, seed=11)
    model = tfm.quantize_model(model, 8)
    model = lowrank.attach_adapters(model, r=8, targets=MATS + ("wh",), seed=7)
    trainer.configure_trainable(model, "lora_finetune")
    slots = {f"layers.{l.index}.{k}": m for l in model.layers for k, m in l.matrices().items()}
    slots["head"] = model.head
    arrays = {"embed": model.embed.weight.data.astype(np.float32)}
    for i, (path, ad) in enumerate(sorted(slots.items())):
        ad.up.data = linalg.seeded_random(*ad.up.data.shape, 500 + i, std=0.02).astype(np.float32)
        q = ad.base.q
        arrays[f"{path}.codes"] = q.codes
        arrays[f"{path}.scale"] = q.scale
        arrays[f"{path}.offset"] = q.offset
        arrays[f"{path}.down"] = ad.down.data
        arrays[f"{path}.up"] = ad.up.data
    rng = np.random.default_rng(13)
    tokens = rng.integers(0, cfg.vocab, size=(2, cfg.max_seq))
    targets = rng.integers(0, cfg.vocab, size=(2, cfg.max_seq))
    logits, tape = tfm.model_forward(model, tokens, tfm.PER_LAYER)
    loss = tfm.cross_entropy_loss(logits, targets)
    grads = tfm.model_backward(model, tape, tfm.cross_entropy_grad(logits, targets))
    assert sorted(grads) == sorted(model.trainable_parameters())
    arrays["tokens"] = tokens
    arrays["targets"] = targets
    arrays["loss"] = np.array(loss)
    for k, g in grads.items():
        arrays[f"grad::{k}"] = g.astype(np.float32)
    arrays["config"] = np.array([cfg.vocab, cfg.dim, cfg.heads, cfg.layers, cfg.ffn_dim, cfg.max_seq])
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, "decoder_small.npz"), **arrays)
    print(f"loss {loss:.6f}, {len(grads)} gradient tensors")


if __name__ == "__main__":
    main()
