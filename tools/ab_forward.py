"""A/B bit comparison of the library's forward output across two builds (development tool).

    QADAPTER_LIB=<lib> python tools/ab_forward.py OUT.pt [--N 4096 --K 4096 --T 16384 --bits 8 --rank 8]

Writes y (and, with --probe, nothing else) for a fixed seed so two builds' outputs can be compared bit for bit.
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
    ap.add_argument("out")
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--T", type=int, default=16384)
    ap.add_argument("--bits", type=int, default=8)
    ap.add_argument("--rank", type=int, default=8)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _lib.lib()
    g = torch.Generator(device=dev).manual_seed(7)
    q = quantize_rows(torch.randn((a.N, a.K), generator=g, device=dev) * 0.02, a.bits)
    spec = TTSpec.for_shape(a.N, a.K, a.rank)
    cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.1 for i in range(spec.d)]
    wc, ttc = q.as_c(), spec.as_c(cores)
    nb = lib.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc), a.T)
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    x = torch.randn((a.T, a.K), generator=g, device=dev).to(torch.bfloat16)
    y = torch.empty((a.T, a.N), dtype=torch.bfloat16, device=dev)
    sptr = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.qa_linear_forward(ctypes.byref(wc), ctypes.byref(ttc), x.data_ptr(), _lib.QA_BF16, a.T,
                                     y.data_ptr(), None, None, None, ws.data_ptr(), nb, sptr), "fwd")
    torch.cuda.synchronize()
    torch.save(y.cpu(), a.out)
    print(a.out, float(y.float().abs().mean()))


if __name__ == "__main__":
    main()
