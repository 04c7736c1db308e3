"""Device timeline of one decode step (the bench's 7-linear 7B set, q/k/v and up/gate as groups, CUDA-graph
replay): CUPTI kernel start / end stamps from torch.profiler, printed relative to the step's first kernel, so
prologue latency, matrix-vector durations and the gaps between launches can be read off directly.
    python tools/decode_timeline.py [T]"""
import ctypes
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2402_13533_b200 import _lib  # noqa: E402
from paper_2402_13533_b200.linear import TTSpec  # noqa: E402
from paper_2402_13533_b200.quant import quantize_rows  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1
SHAPES = [("wq", 4096, 4096), ("wk", 4096, 4096), ("wv", 4096, 4096), ("wo", 4096, 4096),
          ("wu", 11008, 4096), ("wg", 11008, 4096), ("wd", 4096, 11008)]
GROUPS = [(0, 1, 2), (3,), (4, 5), (6,)]
dev = torch.device("cuda", 0)
lib = _lib.lib()
g = torch.Generator(device=dev).manual_seed(1)
mats = []
for name, N, K in SHAPES:
    q = quantize_rows(torch.randn((N, K), generator=g, device=dev) * 0.02, 8)
    spec = TTSpec.for_shape(N, K, 8)
    cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
    mats.append((q, cores, q.as_c(), spec.as_c(cores), torch.randn((T, K), generator=g, device=dev).to(torch.bfloat16),
                 torch.empty((T, N), dtype=torch.bfloat16, device=dev)))
nb = 0
gsets = []
for gi in GROUPS:
    n = len(gi)
    W = (ctypes.POINTER(_lib.QWeight) * n)(*[ctypes.pointer(mats[i][2]) for i in gi])
    Tt = (ctypes.POINTER(_lib.TT) * n)(*[ctypes.pointer(mats[i][3]) for i in gi])
    Y = (ctypes.c_void_p * n)(*[mats[i][5].data_ptr() for i in gi])
    nb = max(nb, lib.qa_group_workspace_bytes(n, W, Tt, T))
    gsets.append((n, W, Tt, Y, mats[gi[0]][4]))
ws = torch.empty(nb, dtype=torch.uint8, device=dev)


def step(sp):
    for n, W, Tt, Y, x in gsets:
        _lib.check(lib.qa_group_forward(n, W, Tt, x.data_ptr(), 1, T, Y, None, None, ws.data_ptr(), nb, sp), "group")


gs = torch.cuda.Stream(dev)
for _ in range(3):
    step(torch.cuda.current_stream(dev).cuda_stream)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=gs):
    step(gs.cuda_stream)
for _ in range(10):
    graph.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
per = len(ev) // 5
last = ev[-per:]
t0 = last[0]["ts"]
for e in last:
    name = e["name"].replace("qa::(anonymous namespace)::", "").replace("void ", "").split("(")[0]
    print(f"{e['ts'] - t0:8.2f} .. {e['ts'] + e['dur'] - t0:8.2f}  ({e['dur']:6.2f} us)  {name}")
print(f"step span {last[-1]['ts'] + last[-1]['dur'] - t0:.2f} us; previous step ended "
      f"{t0 - (ev[-per - 1]['ts'] + ev[-per - 1]['dur']):.2f} us before this one began")
