"""Generate tests/golden/*.npz by running the REFERENCE package itself (lrlm).

Run in the build container only (it needs /root/reference, which does not exist on
the GPU box):

    python oracle/gen_golden.py            # writes tests/golden/*.npz

The fixtures pin the oracle restatement (oracle/qa_oracle.py) to the reference's
own outputs on seeded inputs: quantize_rows / dequantize_rows / qmatmul /
qmatmul_t / quantize_activations (quant.py), LoraLinear over QuantizedLinear
forward+backward (transformer.py:246-327), lora_merge (lowrank.py:245-257),
seeded_random (linalg.py:127-152), plus the KAT inputs of pkg/tests/test_quant.py.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = os.environ.get("LRLM_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    sys.path.insert(0, REF)
    from lrlm import linalg, lowrank, quant  # noqa: E402  (reference, read-only)
    from lrlm import transformer as tfm  # noqa: E402

    os.makedirs(OUT, exist_ok=True)

    # 1. quantize_rows cases: (name, grid) for bits 4 and 8.
    cases = {
        "ongrid": np.array([[0.0, 1.0, 2.0, 3.0]], dtype=np.float32),  # test_quant.py:26-29
        "const": np.full((3, 5), 2.5, dtype=np.float32),  # test_quant.py:19-24
        "zeros": np.zeros((4, 6), dtype=np.float32),
        "extremes": linalg.seeded_random(12, 17, seed=6),  # test_quant.py:59-70
        "odd4": linalg.seeded_random(3, 7, seed=9),  # test_quant.py:81-86
        "uniform": linalg.seeded_random(64, 32, seed=8, dist="uniform", lo=-3, hi=5),  # test_quant.py:31-37
        "gauss": linalg.seeded_random(37, 53, seed=11, std=0.02),
        "wide": linalg.seeded_random(5, 1031, seed=12),
        # exact half-way values: (w - lo)/scale lands on k + 0.5 -> ties away from zero
        "ties": (np.arange(0, 511, dtype=np.float32)[None, :] * 0.5).repeat(2, 0),
        # near-ties: half-integers perturbed by one f32 ulp either side
        "nearties": np.stack([
            np.concatenate([[0.0], np.nextafter(np.arange(1, 255, dtype=np.float32) + 0.5, np.float32(0)), [255.0]]),
            np.concatenate([[0.0], np.nextafter(np.arange(1, 255, dtype=np.float32) + 0.5, np.float32(1e9)), [255.0]]),
        ]).astype(np.float32),
        "negconst": np.tile(np.array([[1.5], [-2.0]], dtype=np.float32), (1, 4)),
    }
    # bf16-valued activations (the GPU path's input dtype), ragged width
    rng = np.random.default_rng(1234)
    act = rng.standard_normal((29, 96)).astype(np.float32)
    act_bits = act.view(np.uint32)
    act = ((act_bits + 0x7FFF + ((act_bits >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)
    cases["act_bf16"] = act

    quant_fix = {}
    for name, w in cases.items():
        quant_fix[f"{name}__w"] = w
        for bits in (4, 8):
            q = quant.quantize_rows(w, bits)
            quant_fix[f"{name}__b{bits}__codes"] = q.codes
            quant_fix[f"{name}__b{bits}__scale"] = q.scale
            quant_fix[f"{name}__b{bits}__offset"] = q.offset
            quant_fix[f"{name}__b{bits}__deq"] = quant.dequantize_rows(q, np.float64)
    np.savez_compressed(os.path.join(OUT, "quant_cases.npz"), **quant_fix)

    # 2. qmatmul / qmatmul_t on small shapes (test_quant.py:101-126 pattern)
    mm = {}
    for bits in (4, 8):
        q = quant.quantize_rows(linalg.seeded_random(9, 13, seed=bits + 10), bits)
        xs = linalg.seeded_random(3, 13, seed=99)
        dy = linalg.seeded_random(3, 9, seed=98)
        mm[f"b{bits}__w"] = linalg.seeded_random(9, 13, seed=bits + 10)
        mm[f"b{bits}__x"] = xs
        mm[f"b{bits}__dy"] = dy
        mm[f"b{bits}__qmatmul"] = quant.qmatmul(q, xs.astype(np.float64))
        mm[f"b{bits}__qmatmul_t"] = quant.qmatmul_t(q, dy.astype(np.float64))
    np.savez_compressed(os.path.join(OUT, "qmatmul_cases.npz"), **mm)

    # 3. LoraLinear over a QuantizedLinear base: forward/backward/merge (anchors the d=2 TT oracle)
    lo = {}
    for bits in (4, 8):
        w = linalg.seeded_random(24, 40, seed=21 + bits, std=0.02)
        down = linalg.seeded_random(4, 40, seed=31 + bits, std=0.02)
        up = linalg.seeded_random(24, 4, seed=41 + bits, std=0.02)
        x = linalg.seeded_random(6, 40, seed=51 + bits).astype(np.float64)
        dy = linalg.seeded_random(6, 24, seed=61 + bits).astype(np.float64)
        base = tfm.QuantizedLinear("w.base", quant.quantize_rows(w, bits))
        ad = tfm.LoraLinear("w", base, down.astype(np.float64), up.astype(np.float64))
        y = ad.forward(x)
        grads = {}
        dx = ad.backward(x, dy, grads)
        lo[f"b{bits}__w"] = w
        lo[f"b{bits}__down"] = down
        lo[f"b{bits}__up"] = up
        lo[f"b{bits}__x"] = x
        lo[f"b{bits}__dy"] = dy
        lo[f"b{bits}__y"] = y
        lo[f"b{bits}__dx"] = dx
        lo[f"b{bits}__gdown"] = grads["w.down"]
        lo[f"b{bits}__gup"] = grads["w.up"]
        # merge onto a dense base (the only merge the reference allows) ...
        dense = tfm.DenseLinear("w.base", w.astype(np.float64), trainable=False)
        ad2 = tfm.LoraLinear("w", dense, down.astype(np.float64), up.astype(np.float64))
        lo[f"b{bits}__merged_dense"] = lowrank.lora_merge(ad2)
        # ... and the reference's refusal to merge onto a quantised base (lowrank.py:249-252)
        try:
            lowrank.lora_merge(ad)
            lo[f"b{bits}__merge_q_refused"] = np.array(0)
        except tfm.ModelError:
            lo[f"b{bits}__merge_q_refused"] = np.array(1)
    np.savez_compressed(os.path.join(OUT, "lora_cases.npz"), **lo)

    # 4. BASELINE config 1 (the oracle/parity config): W 1024^2 ~N(0,0.02) int8, x [4,128,1024] ~N(0,1)
    W = linalg.seeded_random(1024, 1024, seed=1, std=0.02)
    X = linalg.seeded_random(512, 1024, seed=2)
    qw = quant.quantize_rows(W, 8)
    qx = quant.quantize_rows(X, 8)  # per-token act-quant = quantize_rows on [T, K]
    qw4 = quant.quantize_rows(W, 4)
    y1 = quant.qmatmul(qw, quant.dequantize_rows(qx, np.float64)[:16])
    dy = linalg.seeded_random(16, 1024, seed=7)
    dxb = quant.qmatmul_t(qw, dy.astype(np.float64))
    c1 = {
        "w_digest": np.array(_digest(W)),
        "x_digest": np.array(_digest(X)),
        "qw_codes_digest": np.array(_digest(qw.codes)),
        "qw4_codes_digest": np.array(_digest(qw4.codes)),
        "qx_codes_digest": np.array(_digest(qx.codes)),
        "qw_scale": qw.scale, "qw_offset": qw.offset,
        "qw4_scale": qw4.scale, "qw4_offset": qw4.offset,
        "qx_scale": qx.scale, "qx_offset": qx.offset,
        "y1_first16": y1,
        "dy_first16": dy,
        "dx_base_first16": dxb,
    }
    np.savez_compressed(os.path.join(OUT, "config1.npz"), **c1)

    # 5. seeded_random stream pins
    sr = {}
    for seed in (0, 1, 7919, 123456789):
        sr[f"g{seed}"] = linalg.seeded_random(3, 5, seed=seed)
        sr[f"u{seed}"] = linalg.seeded_random(2, 7, seed=seed, dist="uniform", lo=-1, hi=2)
    np.savez_compressed(os.path.join(OUT, "seeded_random.npz"), **sr)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
