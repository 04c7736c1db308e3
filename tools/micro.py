"""Per-kernel-class timing of one quantised adapter linear (development micro-benchmark).

    python tools/micro.py [--N 4096] [--K 4096] [--T 16384] [--bits 8] [--rank 8] [--iters 20] [--only fwd|bwd]

Prints, per call, the device time of each kernel class (library CUDA-event timing) and the
algorithmic rate.  Run under ncu with -k regex:<kernel> to profile one kernel in isolation.
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402
from paper_2402_13533_b200.linear import TTSpec  # noqa: E402
from paper_2402_13533_b200.quant import quantize_rows  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--bits", type=int, default=8)
    ap.add_argument("--rank", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", choices=["fwd", "bwd", "both"], default="both")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _lib.lib()
    g = torch.Generator(device=dev).manual_seed(1)
    q = quantize_rows(torch.randn((a.N, a.K), generator=g, device=dev) * 0.02, a.bits)
    spec = TTSpec.for_shape(a.N, a.K, a.rank if a.rank > 0 else 8)
    cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
    wc = q.as_c()
    ttc = spec.as_c(cores) if a.rank > 0 else None  # --rank 0: the base linear alone (no adapter)
    ttp = ctypes.byref(ttc) if ttc is not None else None
    nb = lib.qa_linear_workspace_bytes(ctypes.byref(wc), ttp, a.T)
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    x = torch.randn((a.T, a.K), generator=g, device=dev).to(torch.bfloat16)
    dy = torch.randn((a.T, a.N), generator=g, device=dev).to(torch.bfloat16)
    y = torch.empty((a.T, a.N), dtype=torch.bfloat16, device=dev)
    dx = torch.empty((a.T, a.K), dtype=torch.bfloat16, device=dev)
    grads = [torch.empty(spec.core_shape(i), device=dev) for i in range(spec.d)]
    gptr = (ctypes.c_void_p * _lib.QA_TT_MAX_D)(*[t.data_ptr() for t in grads])
    sptr = torch.cuda.current_stream(dev).cuda_stream

    def run():
        if a.only in ("fwd", "both"):
            _lib.check(lib.qa_linear_forward(ctypes.byref(wc), ttp, x.data_ptr(), _lib.QA_BF16, a.T,
                                             y.data_ptr(), None, None, None, ws.data_ptr(), nb, sptr), "fwd")
        if a.only in ("bwd", "both"):
            _lib.check(lib.qa_linear_backward(ctypes.byref(wc), ttp, x.data_ptr(), _lib.QA_BF16,
                                              dy.data_ptr(), _lib.QA_BF16, a.T, dx.data_ptr(), None,
                                              ctypes.cast(gptr, ctypes.POINTER(ctypes.c_void_p)), 0, ws.data_ptr(),
                                              nb, sptr), "bwd")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    lib.qa_timing_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / a.iters
    print(f"N={a.N} K={a.K} T={a.T} bits={a.bits} r={a.rank} only={a.only}: {total * 1e3:.1f} us per call")
    for c in ("gemm_i8", "gemm_bf16", "quantize", "tt", "dequant"):
        ms, n, work = _lib.timing_read(c)
        if n == 0:
            continue
        per = ms / n * 1e3
        unit = "TOPS" if c.startswith("gemm") else ("GB/s" if c != "tt" else "TFLOP/s")
        rate = work / n / (ms / n / 1e3) / (1e12 if unit != "GB/s" else 1e9)
        print(f"  {c:10s} {ms / a.iters * 1e3:8.1f} us/call  {n // a.iters:3d} launches  {per:7.1f} us/launch  "
              f"{rate:8.1f} {unit}")
    lib.qa_timing_enable(0)


if __name__ == "__main__":
    main()
