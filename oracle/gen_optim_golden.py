"""Generate tests/golden/adamw.npz with the REFERENCE optimizer (trainer.py:84-121 adamw_step).

Test infrastructure only; run in the build container:  python oracle/gen_optim_golden.py
Three tensors of adapter-like shapes, seeded gradients, three steps; the parameters (float32) and the
float64 masters after every step are recorded.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("LRLM_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from lrlm import linalg, trainer  # noqa: E402  (reference, read-only)
    from lrlm import transformer as tfm  # noqa: E402

    shapes = {"layers.0.wq.core0": (1, 1, 16, 8), "layers.0.wq.core1": (8, 4, 4, 8), "layers.0.wq.core2": (8, 256, 1, 1)}
    params = {}
    for i, (k, shp) in enumerate(sorted(shapes.items())):
        n = int(np.prod(shp))
        params[k] = tfm.Param(k, linalg.seeded_random(1, n, 10 + i, std=0.01).astype(np.float32).reshape(shp))
    cfg = trainer.TrainConfig(lr=1e-3, weight_decay=0.05)
    state = trainer.AdamWState(params)
    out = {}
    for k, p in params.items():
        out[f"init__{k}"] = p.data.copy()
    for t in range(3):
        grads = {}
        for i, (k, p) in enumerate(sorted(params.items())):
            grads[k] = linalg.seeded_random(1, p.data.size, 100 * t + i, std=0.1).astype(np.float32).reshape(p.data.shape)
            out[f"g{t}__{k}"] = grads[k]
        trainer.adamw_step(state, params, grads, cfg)
        for k, p in params.items():
            out[f"p{t}__{k}"] = p.data.copy()
            out[f"w{t}__{k}"] = state.master[k].copy()
    np.savez_compressed(os.path.join(OUT, "adamw.npz"), **out)
    print("wrote", os.path.join(OUT, "adamw.npz"))


if __name__ == "__main__":
    main()
