"""Phase timestamps (globaltimer, ns) of the decode prologue k_decode_prep, from a -DQA_DP_TRACE build:
    python -m paper_2402_13533_b200.build -DQA_DP_TRACE --out=paper_2402_13533_b200/libqadapter_trace.so
    QADAPTER_LIB=paper_2402_13533_b200/libqadapter_trace.so python tools/decode_trace.py [K] [N]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402
from paper_2402_13533_b200.linear import TTSpec  # noqa: E402
from paper_2402_13533_b200.quant import quantize_rows  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dev = torch.device("cuda", 0)
lib = _lib.lib()
g = torch.Generator(device=dev).manual_seed(1)
q = quantize_rows(torch.randn((N, K), generator=g, device=dev) * 0.02, 8)
spec = TTSpec.for_shape(N, K, 8)
cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
wc, ttc = q.as_c(), spec.as_c(cores)
nb = lib.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc), 1)
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
x = torch.randn((1, K), generator=g, device=dev).to(torch.bfloat16)
y = torch.empty((1, N), dtype=torch.bfloat16, device=dev)
s = torch.cuda.current_stream(dev).cuda_stream
f = lib.qa_debug_dp_trace
f.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 16)()
for it in range(6):
    lib.qa_linear_forward(ctypes.byref(wc), ctypes.byref(ttc), x.data_ptr(), 1, 1, y.data_ptr(), None, None, None,
                          ws.data_ptr(), nb, s)
    torch.cuda.synchronize()
    f(buf)
    t0 = buf[0]
    print(f"K={K} N={N} it{it}: " + " ".join(f"{i}:{(buf[i] - t0) / 1e3:.2f}" for i in range(1, 10) if buf[i] >= t0))
