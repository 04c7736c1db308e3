"""Measure a library int8 tensor-core reference peak on this B200 (cuBLASLt through torch._int_mm).

MEASURED_PEAKS.json (driver-written) has HBM copy and bf16 GEMM peaks but no int8 figure, so the
int8 GEMM's roofline fraction is reported against this measured library number (and the 4.5 POPS
spec for context).  Writes profiles/int8_peak.json.

    python tools/measure_int8_peak.py
"""

from __future__ import annotations

import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(m, n, k, iters=10):
    a = torch.randint(-128, 127, (m, k), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, k), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    # sustained: back to back for ~3 s
    t_end = time.time() + 3.0
    n_it = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() < t_end:
        for _ in range(20):
            torch._int_mm(a, b)
        n_it += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / 1e3 / n_it
    ops = 2.0 * m * n * k
    return ops / best / 1e12, ops / sus / 1e12


def main():
    out = {"how": "torch._int_mm (cuBLASLt s8 x s8 -> s32), best of 10 (burst) and back to back for 3 s "
                  "(sustained), CUDA events", "gpu": torch.cuda.get_device_name(0), "shapes": {}}
    best_burst = best_sus = 0.0
    for (m, n, k) in [(16384, 4096, 4096), (16384, 11008, 4096), (8192, 8192, 8192)]:
        burst, sus = bench(m, n, k)
        out["shapes"][f"{m}x{n}x{k}"] = {"burst_tops": burst, "sustained_tops": sus}
        best_burst, best_sus = max(best_burst, burst), max(best_sus, sus)
    out["int8_tops"] = best_burst
    out["int8_tops_sustained"] = best_sus
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "int8_peak.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
