"""Throughput of the merge kernel (qa_merge: W' = dequantize_rows(q) + W_t, lowrank.py:245-257) on the
BASELINE config-5 shapes (Llama-2-70B linears, int4, TT r = 8) and the 7B set (int8).

    python tools/merge_bench.py [--set 70b|7b] [--out bf16|f32] [--iters 10]

Prints one JSON line: per-matrix and total algorithmic bytes (codes in + W' out), device
time (CUDA events, warm), GB/s and the fraction of the measured HBM copy peak.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402
from paper_2402_13533_b200.linear import TTSpec  # noqa: E402
from paper_2402_13533_b200.quant import quantize_rows  # noqa: E402

SETS = {
    "70b": [("wq", 8192, 8192), ("wk", 1024, 8192), ("wv", 1024, 8192), ("wo", 8192, 8192),
            ("wu", 28672, 8192), ("wg", 28672, 8192), ("wd", 8192, 28672)],
    "7b": [("wq", 4096, 4096), ("wk", 4096, 4096), ("wv", 4096, 4096), ("wo", 4096, 4096),
           ("wu", 11008, 4096), ("wg", 11008, 4096), ("wd", 4096, 11008)],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", choices=sorted(SETS), default="70b")
    ap.add_argument("--out", choices=["bf16", "f32"], default="bf16")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    bits = 4 if a.set == "70b" else 8
    dev = torch.device("cuda", 0)
    lib = _lib.lib()
    g = torch.Generator(device=dev).manual_seed(5)
    odt = torch.bfloat16 if a.out == "bf16" else torch.float32
    sptr = torch.cuda.current_stream(dev).cuda_stream
    rows, tot_bytes, tot_ms = [], 0.0, 0.0
    for name, n, k in SETS[a.set]:
        q = quantize_rows(torch.randn((n, k), generator=g, device=dev) * 0.02, bits)
        spec = TTSpec.for_shape(n, k, 8)
        cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
        wc, ttc = q.as_c(), spec.as_c(cores)
        nb = lib.qa_merge_workspace_bytes(ctypes.byref(ttc))
        ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)
        out = torch.empty((n, k), dtype=odt, device=dev)

        def run():
            _lib.check(lib.qa_merge(ctypes.byref(wc), ctypes.byref(ttc), out.data_ptr(),
                                    _lib.QA_BF16 if a.out == "bf16" else _lib.QA_F32, ws.data_ptr(), ws.numel(),
                                    sptr), "qa_merge")

        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        byts = n * k * bits / 8 + n * k * out.element_size() + 8 * n + 4 * spec.param_count()
        rows.append({"name": name, "shape": [n, k], "ms": ms, "gbs": byts / ms / 1e6})
        tot_bytes += byts
        tot_ms += ms
        del q, out, ws
    peak = None
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p)).get("hbm_gbs")
    gbs = tot_bytes / tot_ms / 1e6
    print(json.dumps({"kernel": "merge (k_merge_fast)", "set": a.set, "bits": bits, "out": a.out,
                      "total_ms": tot_ms, "total_bytes": tot_bytes, "achieved_gbs": gbs,
                      "frac_of_hbm": gbs / peak if peak else None, "per_matrix": rows}))


if __name__ == "__main__":
    main()
