"""Decode step (1 / 8 tokens through the 7-linear 7B set) kernel breakdown: CUDA-event step time and the warm
per-kernel durations from torch.profiler (CUPTI), to split prologue / matrix-vector / gaps.

    python tools/decode_profile.py [T]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402
from paper_2402_13533_b200.linear import TTSpec  # noqa: E402
from paper_2402_13533_b200.quant import quantize_rows  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1
SHAPES = [("wq", 4096, 4096), ("wk", 4096, 4096), ("wv", 4096, 4096), ("wo", 4096, 4096),
          ("wu", 11008, 4096), ("wg", 11008, 4096), ("wd", 4096, 11008)]
dev = torch.device("cuda", 0)
lib = _lib.lib()
g = torch.Generator(device=dev).manual_seed(1)
mats = []
nb = 0
for name, N, K in SHAPES:
    q = quantize_rows(torch.randn((N, K), generator=g, device=dev) * 0.02, 8)
    spec = TTSpec.for_shape(N, K, 8)
    cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
    wc, ttc = q.as_c(), spec.as_c(cores)
    nb = max(nb, lib.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc), T))
    x = torch.randn((T, K), generator=g, device=dev).to(torch.bfloat16)
    y = torch.empty((T, N), dtype=torch.bfloat16, device=dev)
    mats.append((q, cores, wc, ttc, x, y))
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream(dev).cuda_stream


GROUP = "--group" in sys.argv
GROUPS = [(0, 1, 2), (3,), (4, 5), (6,)]  # q/k/v and up/gate share their input
gsets = []
for gi in GROUPS:
    n = len(gi)
    W = (ctypes.POINTER(_lib.QWeight) * n)(*[ctypes.pointer(mats[i][2]) for i in gi])
    Tt = (ctypes.POINTER(_lib.TT) * n)(*[ctypes.pointer(mats[i][3]) for i in gi])
    Y = (ctypes.c_void_p * n)(*[mats[i][5].data_ptr() for i in gi])
    nb = max(nb, lib.qa_group_workspace_bytes(n, W, Tt, T))
    gsets.append((n, W, Tt, Y, mats[gi[0]][4]))
ws = torch.empty(nb, dtype=torch.uint8, device=dev)


def step():
    if GROUP:
        for n, W, Tt, Y, x in gsets:
            _lib.check(lib.qa_group_forward(n, W, Tt, x.data_ptr(), 1, T, Y, None, None, ws.data_ptr(), nb, s),
                       "group forward")
        return
    for q, cores, wc, ttc, x, y in mats:
        _lib.check(lib.qa_linear_forward(ctypes.byref(wc), ctypes.byref(ttc), x.data_ptr(), 1, T, y.data_ptr(), None,
                                          None, None, ws.data_ptr(), nb, s), "forward")


for _ in range(20):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    step()
e1.record()
torch.cuda.synchronize()
print(f"T={T}: {e0.elapsed_time(e1) / 100 * 1e3:.1f} us per 7-linear step (CUDA events)")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        step()
    torch.cuda.synchronize()
tot = 0.0
for ev in prof.key_averages():
    if ev.device_type.name == "CUDA" and ev.count:
        us = ev.device_time_total / 20
        tot += us
        print(f"  {us:8.1f} us/step  {ev.count // 20:3d}/step  avg {ev.device_time_total / ev.count:6.2f} us  {ev.key[:90]}")
print(f"  kernel sum {tot:.1f} us/step")
