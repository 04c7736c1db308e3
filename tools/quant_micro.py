"""Weight quantiser in isolation (for ncu): qa_quantize_rows over the 7B shapes (f32 -> int8) and the 70B gate / q
shapes (f32 -> int4), a few warm launches each.   python tools/quant_micro.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.lib()
s = torch.cuda.current_stream(dev).cuda_stream
g = torch.Generator(device=dev).manual_seed(3)
for n, k, bits in ((4096, 4096, 8), (11008, 4096, 8), (4096, 11008, 8), (28672, 8192, 4), (8192, 8192, 4)):
    w = torch.randn((n, k), generator=g, device=dev) * 0.02
    ld = k if bits == 8 else (k + 1) // 2
    codes = torch.empty((n, ld), dtype=torch.uint8, device=dev)
    sc, of = torch.empty(n, device=dev), torch.empty(n, device=dev)
    rs = torch.empty(n, dtype=torch.int32, device=dev)
    for _ in range(3):
        _lib.check(lib.qa_quantize_rows(w.data_ptr(), _lib.QA_F32, n, k, k, bits, codes.data_ptr(), ld, k,
                                        sc.data_ptr(), of.data_ptr(), rs.data_ptr(), None, s), "quantize")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _lib.check(lib.qa_quantize_rows(w.data_ptr(), _lib.QA_F32, n, k, k, bits, codes.data_ptr(), ld, k,
                                        sc.data_ptr(), of.data_ptr(), rs.data_ptr(), None, s), "quantize")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byts = n * k * 4 + n * ld + 12 * n
    print(f"{n}x{k} int{bits}: {ms * 1e3:.1f} us, {byts / ms / 1e6:.0f} GB/s")
