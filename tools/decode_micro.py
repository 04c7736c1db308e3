"""Decode-step kernels in isolation (for ncu): 1..8 tokens through one 4096x4096 adapter linear."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402
from paper_2402_13533_b200.linear import TTSpec  # noqa: E402
from paper_2402_13533_b200.quant import quantize_rows  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = K = 4096
dev = torch.device("cuda", 0)
lib = _lib.lib()
g = torch.Generator(device=dev).manual_seed(1)
q = quantize_rows(torch.randn((N, K), generator=g, device=dev) * 0.02, 8)
spec = TTSpec.for_shape(N, K, 8)
cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
wc, ttc = q.as_c(), spec.as_c(cores)
nb = lib.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc), T)
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
x = torch.randn((T, K), generator=g, device=dev).to(torch.bfloat16)
y = torch.empty((T, N), dtype=torch.bfloat16, device=dev)
s = torch.cuda.current_stream(dev).cuda_stream
for _ in range(20):
    lib.qa_linear_forward(ctypes.byref(wc), ctypes.byref(ttc), x.data_ptr(), 1, T, y.data_ptr(), None, None, None,
                          ws.data_ptr(), nb, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    lib.qa_linear_forward(ctypes.byref(wc), ctypes.byref(ttc), x.data_ptr(), 1, T, y.data_ptr(), None, None, None,
                          ws.data_ptr(), nb, s)
e1.record()
torch.cuda.synchronize()
print(f"T={T}: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us per forward")
