"""Generate tests/golden/ckpt_small.lrlm (+ ckpt_small.npz) with the REFERENCE package (lrlm).

Test infrastructure only; run in the build container (it needs /root/reference):

    python oracle/gen_checkpoint_golden.py

A one-layer model with int8 attention / head and int4 FFN bases (quantize_model,
transformer.py:1114-1133) and LoRA adapters on wq / wv / wu (attach_adapters, lowrank.py:189-234,
with the zero-initialised `up` factors replaced by seeded values) is written by the reference's own
save_checkpoint (checkpoint.py:113-140).  The npz holds the arrays the reference holds in memory, so
the device loader (paper_2402_13533_b200/checkpoint.py) is pinned to the reference's layout
(u8q / u4q packed codes, checkpoint.py:64-70) and its writer to byte-identical output.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("LRLM_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from lrlm import checkpoint, linalg, lowrank  # noqa: E402  (reference, read-only)
    from lrlm import transformer as tfm  # noqa: E402

    cfg = tfm.ModelConfig(vocab=64, dim=64, heads=2, layers=1, ffn_dim=96, max_seq=16)
    model = tfm.build_model(cfg, seed=3)
    model = tfm.quantize_model(model, 8, ("wq", "wk", "wv", "wo", "wh"))
    model = tfm.quantize_model(model, 4, ("wu", "wg", "wd"))
    model = lowrank.attach_adapters(model, r=4, targets=("wq", "wv", "wu"), seed=5)
    arrays = {}
    layer = model.layers[0]
    for i, name in enumerate(("wq", "wv", "wu")):
        ad = getattr(layer, name)
        ad.up.data = linalg.seeded_random(*ad.up.data.shape, 100 + i, std=0.02).astype(np.float32)
        arrays[f"{name}.down"] = ad.down.data
        arrays[f"{name}.up"] = ad.up.data
        q = ad.base.q
        arrays[f"{name}.codes"], arrays[f"{name}.scale"], arrays[f"{name}.offset"] = q.codes, q.scale, q.offset
        arrays[f"{name}.bits"] = np.array(q.bits)
    for name in ("wk", "wo", "wg", "wd"):
        q = getattr(layer, name).q
        arrays[f"{name}.codes"], arrays[f"{name}.scale"], arrays[f"{name}.offset"] = q.codes, q.scale, q.offset
        arrays[f"{name}.bits"] = np.array(q.bits)
    path = os.path.join(OUT, "ckpt_small.lrlm")
    checkpoint.save_checkpoint(path, model)
    np.savez_compressed(os.path.join(OUT, "ckpt_small.npz"), **arrays)
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
