"""Kernel-time breakdown of one decoder step (torch.profiler / CUPTI) — which kernels the glue costs.

    python tools/decoder_profile.py [--layers 2] [--batch 4] [--seq 2048]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2402_13533_b200.decoder import DecoderConfig, build_decoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--seq", type=int, default=2048)
a = ap.parse_args()
cfg = DecoderConfig(vocab=32000, dim=4096, heads=32, layers=a.layers, ffn_dim=11008, max_seq=a.seq)
model = build_decoder(cfg, rank=8, bits=8, seed=1)
tok = torch.randint(0, cfg.vocab, (a.batch, a.seq), device="cuda")
for _ in range(2):
    model.train_step_grads(tok, tok)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    model.train_step_grads(tok, tok)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=90))
