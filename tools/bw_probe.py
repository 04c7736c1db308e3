"""HBM probes on the box: write-only, read-only and copy bandwidth with plain torch ops (the ceilings the
merge (80% writes) and quantise (80% reads) kernels are judged against), CUDA events, best of N."""
import json
import sys

import torch


def best(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


def main():
    n = 1 << 30  # 1 Gi bf16 elements = 2 GiB
    x = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    x.normal_()
    r = {}
    ms = best(lambda: y.fill_(1.0))
    r["write_gbs"] = 2 * n / ms / 1e6
    ms = best(lambda: y.copy_(x))
    r["copy_gbs"] = 4 * n / ms / 1e6
    xi = x.view(torch.int32)
    ms = best(lambda: torch.sum(xi, dtype=torch.int64))
    r["read_gbs"] = 2 * n / ms / 1e6
    print(json.dumps(r))


if __name__ == "__main__":
    sys.exit(main())
