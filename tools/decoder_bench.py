"""BASELINE config 4 on one GPU: the 32-layer Llama-2-7B-shaped decoder stack (hidden 4096, 32 heads, FFN 11008,
vocab 32000), int8 bases + TT adapters (r = 8) on every linear and the head, PER_LAYER recompute; 4 x 2048
tokens per GPU (the [32, 2048] global batch over 8 GPUs).  One step = forward storing each layer's input,
cross-entropy, backward re-running each layer, AdamW on the adapter cores (DecoderStack.train_step).

    python tools/decoder_bench.py [--layers 32] [--batch 4] [--seq 2048] [--steps 3] [--warmup 2]

Prints one JSON line: tokens/s, ms/step (CUDA events over the timed steps), peak device memory, last loss.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2402_13533_b200.decoder import DecoderConfig, build_decoder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    cfg = DecoderConfig(vocab=32000, dim=4096, heads=32, layers=a.layers, ffn_dim=11008, max_seq=a.seq)
    torch.cuda.set_device(0)
    model = build_decoder(cfg, rank=8, bits=8, seed=1)
    g = torch.Generator(device="cuda").manual_seed(2)
    tokens = torch.randint(0, cfg.vocab, (a.batch, a.seq), generator=g, device="cuda")
    targets = torch.randint(0, cfg.vocab, (a.batch, a.seq), generator=g, device="cuda")
    state = None
    for _ in range(a.warmup):
        _, state = model.train_step(tokens, targets, state)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = []
    for _ in range(a.steps):
        loss, state = model.train_step(tokens, targets, state)
        losses.append(loss)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    T = a.batch * a.seq
    print(json.dumps({
        "metric": "decoder training step (per-layer recompute + AdamW) tokens/s", "value": T / (ms / 1e3), "unit": "tokens/s",
        "ms_per_step": ms, "steps": a.steps, "warmup": a.warmup, "dtype": "int8 weights x bf16 activations",
        "config": {"workload": f"llama2-7b decoder, {a.layers} layers, vocab 32000, TT r=8 on all linears + head, "
                               f"int8 bases, PER_LAYER recompute, [{a.batch}, {a.seq}] tokens/GPU",
                   "baseline_config": 4},
        "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9, "loss": losses[-1],
        "adapter_tensors": len(state.names)}))


if __name__ == "__main__":
    main()
