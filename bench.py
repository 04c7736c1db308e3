"""Benchmark of the quantised tensor-adapter linear hot path (BASELINE.json north star).

Workload (BASELINE.json configs[1], "config 2"): the Llama-2-7B linear set — q/k/v/o 4096x4096,
gate/up 11008x4096, down 4096x11008 — int8 per-row quantised from ~N(0, 0.02) weights, a TT
adapter of rank 8 on every linear, 8x2048 = 16384 bf16 tokens ~N(0, 1) per GPU.  One step =
forward (per-token act-quant, int8 tcgen05 GEMM, dequant epilogue + adapter) and backward with
recompute (adapter-core gradients + dx) of all seven linears, then (N > 1) the NCCL all-reduce
of the flat adapter-gradient buffer.  Data is synthetic (seeded); there is no dataset.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|3|4]

--config 4 runs the 32-layer decoder training step (per-layer recompute + AdamW, 8192 tokens per GPU) as the
step instead of the linear set.

N > 1 runs under torchrun (one process per GPU, NCCL); the line is printed by rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quantized-adapter linear fwd+bwd tokens/s"
UNIT = "tokens/s"

LINEARS_7B = [  # (name, fan_out, fan_in, input) in forward order (transformer.py:862-874)
    ("wq", 4096, 4096, "attn"), ("wk", 4096, 4096, "attn"), ("wv", 4096, 4096, "attn"),
    ("wo", 4096, 4096, "ctx"), ("wu", 11008, 4096, "ffn"), ("wg", 11008, 4096, "ffn"),
    ("wd", 4096, 11008, "act"),
]
LINEARS_70B = [  # config 5: hidden 8192, FFN 28672, GQA 8 KV heads of 128 (k / v project to 1024)
    ("wq", 8192, 8192, "attn"), ("wk", 1024, 8192, "attn"), ("wv", 1024, 8192, "attn"),
    ("wo", 8192, 8192, "ctx"), ("wu", 28672, 8192, "ffn"), ("wg", 28672, 8192, "ffn"),
    ("wd", 8192, 28672, "act"),
]
BACKWARD_ORDER = ["wd", "wu", "wg", "wo", "wq", "wk", "wv"]  # transformer.py:919-944
# members that read the same input run as one shared-input group (qa_group_forward / _backward):
# wq / wk / wv on norm1 and wu / wg on norm2 (transformer.py:862-874)
GROUPS_FWD = [("wq", "wk", "wv"), ("wo",), ("wu", "wg"), ("wd",)]
GROUPS_BWD = [("wd",), ("wu", "wg"), ("wo",), ("wq", "wk", "wv")]
INPUT_DIMS = {"attn": 4096, "ctx": 4096, "ffn": 4096, "act": 11008}
INPUT_DIMS_70B = {"attn": 8192, "ctx": 8192, "ffn": 8192, "act": 28672}

CONFIGS = {
    "2": {"bits": 8, "rank": 8, "batch": 8, "seq": 2048},
    "3": {"bits": 4, "rank": 16, "batch": 16, "seq": 4096},  # global tokens; sharded over ranks
    "4": {"bits": 8, "rank": 8, "batch": 4, "seq": 2048},  # decoder stack: 4 sequences per GPU (32 over 8 GPUs)
    "5": {"bits": 4, "rank": 8, "batch": 8, "seq": 4096},  # 70B linear set, [8, 4096] tokens per GPU
}


def linear_set(cfg_name):
    """(linears, input dims) of a config: the 7B set for configs 1-4, the 70B set for config 5."""
    return (LINEARS_70B, INPUT_DIMS_70B) if cfg_name == "5" else (LINEARS_7B, INPUT_DIMS)
DECODER_LAYERS = 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-merge", action="store_true")
    ap.add_argument("--no-decoder", action="store_true", help="skip the config-4 decoder-stack measurement")
    ap.add_argument("--no-group", action="store_true", help="run every linear on its own (A/B of the shared x pass)")
    return ap.parse_args()


def workload_config(cfg_name, world):
    c = CONFIGS[cfg_name]
    if cfg_name == "3":  # [16, 4096] global tokens, strong-scaled over ranks
        tokens = c["batch"] * c["seq"] // world
        scaling = "strong"
    else:
        tokens = c["batch"] * c["seq"]
        scaling = "weak"
    lset = ("llama2-70b linear set q/o 8192x8192, k/v 1024x8192 (GQA), gate/up 28672x8192, down 8192x28672"
            if cfg_name == "5" else "llama2-7b linear set q/k/v/o 4096x4096, gate/up 11008x4096, down 4096x11008")
    desc = {
        "workload": (f"{lset}; int{c['bits']} "
                     f"per-row weights; TT adapter r={c['rank']} m=(1,N/256,256) n=(K/4,4,1); "
                     f"{tokens} bf16 tokens/GPU; fwd + bwd-with-recompute (+ NCCL grad all-reduce); q/k/v and "
                     f"up/gate as shared-input groups (one x pass per direction, transformer.py:862-874)"),
        "baseline_config": int(cfg_name),
        "tokens_per_gpu": tokens,
        "bits": c["bits"],
        "rank": c["rank"],
        "l2": ("inputs larger than L2 (>= 763 MB of layer inputs + 1.4 GB of upstream grads per step)"
               if cfg_name != "5" else "inputs larger than L2 (3.4 GB of layer inputs + 4.8 GB of upstream grads)"),
        "parallelism": f"dp{world}",
    }
    return c, tokens, scaling, desc


def clocks_sampler_start(path):
    try:
        return subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits", "-lms", "200"],
            stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except Exception:
        return None


def clocks_sampler_stop(proc, path, device_index):
    if proc is None:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    proc.terminate()
    try:
        proc.wait(timeout=5)
    except Exception:
        proc.kill()
    sms, maxes, reasons = [], [], set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in open(path):
        parts = [p.strip() for p in line.split(",")]
        if len(parts) < 9 or not parts[0].isdigit() or int(parts[0]) != device_index:
            continue
        try:
            sms.append(float(parts[1]))
            maxes.append(float(parts[2]))
        except ValueError:
            continue
        for nm, flag in zip(names, parts[5:9]):
            if flag.lower() == "active":
                reasons.add(nm)
    return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxes) if maxes else None,
            "reasons": sorted(reasons), "samples": len(sms)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------------------- CPU baseline / reference arm


def cpu_reference_step_fn(cfg, sample_tokens, seed=0, linset=None):
    """The oracle's staged numpy port of the same 7-linear step on `sample_tokens` tokens
    (TEST/BASELINE INFRASTRUCTURE: used only for the CPU baseline and --impl reference)."""
    import numpy as np

    import oracle as O

    LINEARS_7B, INPUT_DIMS = linset or (globals()["LINEARS_7B"], globals()["INPUT_DIMS"])
    rng = np.random.default_rng(seed)
    mats = {}
    for name, n, k, _ in LINEARS_7B:
        w = (rng.standard_normal((n, k), dtype=np.float32) * 0.02)
        q = O.quantize_rows(w, cfg["bits"])
        shape = O.tt_modes_for(n, k, cfg["rank"])
        cores = [rng.standard_normal(shape.core_shape(i)) * 0.01 for i in range(shape.d)]
        mats[name] = (q, cores)
    xs = {kind: O.to_bf16(rng.standard_normal((sample_tokens, d), dtype=np.float32)) for kind, d in INPUT_DIMS.items()}
    dys = {name: O.to_bf16(rng.standard_normal((sample_tokens, n), dtype=np.float32)) for name, n, _, _ in LINEARS_7B}
    inputs = {name: kind for name, _, _, kind in LINEARS_7B}

    def step():
        for name, _, _, _ in LINEARS_7B:
            q, cores = mats[name]
            O.qa_step_staged(xs[inputs[name]], dys[name], q, cores)

    return step


def lrlm_available() -> bool:
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import lrlm  # noqa: F401  (the unmodified reference, pip-installed into baseline/_ref)
    except ImportError:
        return False
    return True


def lrlm_reference_step_fn(cfg_name, sample_tokens, seed=0):
    """The reference's OWN CPU code for the path (lrlm, baseline/_ref), through its public API: per linear,
    quant.quantize_rows on the [T, K] activations (the per-token act-quant the paper adds, quant.py:73-99), then
    transformer.LoraLinear over a QuantizedLinear base (its adapter; transformer.py:276-327) forward on the
    dequantised activations and backward with recompute (qmatmul / qmatmul_t, quant.py:123-144).  Weights are
    quantised outside the timed region."""
    import numpy as np
    from lrlm import linalg, quant
    from lrlm import transformer as tfm

    cfg = CONFIGS[cfg_name]
    linears, dims = linear_set(cfg_name)
    r = cfg["rank"]
    mats = {}
    for i, (name, n, k, _) in enumerate(linears):
        q = quant.quantize_rows(linalg.seeded_random(n, k, seed + 10 * i + 1, std=0.02), cfg["bits"])
        down = linalg.seeded_random(r, k, seed + 10 * i + 2, std=0.02)
        up = linalg.seeded_random(n, r, seed + 10 * i + 3, std=0.02)
        mats[name] = tfm.LoraLinear(name, tfm.QuantizedLinear(name + ".base", q), down, up)
    rng = np.random.default_rng(seed)
    xs = {kind: rng.standard_normal((sample_tokens, d), dtype=np.float32) for kind, d in dims.items()}
    dys = {name: rng.standard_normal((sample_tokens, n), dtype=np.float32) for name, n, _, _ in linears}
    inputs = {name: kind for name, _, _, kind in linears}

    def step():
        grads = {}
        for name, _, _, _ in linears:
            x = xs[inputs[name]]
            xq = quant.dequantize_rows(quant.quantize_rows(x, 8))
            mats[name].forward(xq)
            mats[name].backward(xq, dys[name], grads)

    return step


def reference_cpu_step(cfg_name, sample_tokens):
    """(step, kind, description) of the CPU reference: lrlm itself when baseline/_ref holds it, else the
    oracle's staged numpy port of the same step."""
    if lrlm_available():
        return (lrlm_reference_step_fn(cfg_name, sample_tokens), "reference",
                "lrlm (baseline/_ref, unmodified): quant.quantize_rows per-token act-quant + LoraLinear(QuantizedLinear) "
                f"fwd + bwd at rank {CONFIGS[cfg_name]['rank']} on each linear")
    return (cpu_reference_step_fn(CONFIGS[cfg_name], sample_tokens, linset=linear_set(cfg_name)), "port",
            "oracle staged numpy fp64 port of the reference path (quant.py quantize_rows/qmatmul/qmatmul_t + TT "
            "adapter)")


def cpu_threads():
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        blas = [i for i in info if i.get("internal_api") in ("openblas", "mkl", "blis")]
        if blas:
            return int(blas[0]["num_threads"]), f"{blas[0]['internal_api']} {blas[0].get('version', '')}".strip()
    except Exception:
        pass
    return os.cpu_count() or 1, "numpy BLAS"


def run_cpu_baseline(cfg_name, sample_tokens=256, repeats=3):
    step, kind, what = reference_cpu_step(cfg_name, sample_tokens)
    step()  # warm (BLAS thread start-up, page faults)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times)
    threads, blas = cpu_threads()
    return {
        "value": sample_tokens / sec,
        "unit": UNIT,
        "cores": threads,
        "kind": kind,
        "sample": (f"{sample_tokens} tokens through all 7 linears (fwd + bwd): {what}; median of {repeats}, {blas}, "
                   f"{threads} threads; weights quantised outside the timed region"),
    }


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    if args.config == "4":
        return run_reference_arm_decoder(args)
    cfg, tokens, scaling, desc = workload_config(args.config, world)
    sample = 64 if args.config == "5" else 1024
    step, kind, what = reference_cpu_step(args.config, sample)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    sec = (time.perf_counter() - t0) / max(args.steps, 1)
    threads, blas = cpu_threads()
    value = sample / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": desc,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample} tokens/step through the 7 linears: {what} ({blas})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def decoder_cpu_rate(sample=64, repeats=2):
    """CPU stand-in for config 4 (a 32-layer decoder is hours of numpy per step): the oracle's staged fp64 port
    of one layer's seven linears, forward + recompute-forward + backward (fwd counted twice) on `sample`
    tokens, scaled to 32 layers; attention, norms and the head are left out, so it overstates the CPU."""
    cfg = CONFIGS["2"]
    step = cpu_reference_step_fn(cfg, sample)
    step()
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times) * (4.0 / 3.0) * DECODER_LAYERS
    threads, blas = cpu_threads()
    return {"value": sample / sec, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} tokens through one layer's 7 linears (oracle staged fp64 port, {blas}), fwd + bwd "
                      f"timed and scaled x4/3 (recompute forward) x{DECODER_LAYERS} layers; glue, attention and "
                      f"head omitted (optimistic for the CPU)"}


def decoder_desc(world):
    c = CONFIGS["4"]
    return {"workload": (f"llama2-7b decoder stack (config 4): {DECODER_LAYERS} layers, hidden 4096, 32 heads, FFN "
                         f"11008, vocab 32000, RMSNorm, RoPE, int8 bases + TT r=8 adapters on all linears and the "
                         f"head, PER_LAYER recompute, AdamW on the adapter cores, [{c['batch']}, {c['seq']}] tokens "
                         f"per GPU (the [32, 2048] global batch at 8 GPUs), NCCL all-reduce of the flat adapter "
                         f"gradients"),
            "baseline_config": 4, "tokens_per_gpu": c["batch"] * c["seq"], "bits": 8, "rank": 8,
            "l2": "inputs larger than L2 (per-layer activations of 8192 tokens)", "parallelism": f"dp{world}"}


def run_reference_arm_decoder(args):
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    cpu = decoder_cpu_rate()
    value = cpu["value"]
    line = {"impl": "reference", "metric": "decoder training step tokens/s", "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 8192 / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": decoder_desc(world), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main_decoder(args):
    """--config 4: the decoder training step as the bench step (DecoderStack.train_step), DP over NCCL."""
    import torch
    import torch.distributed as dist

    from paper_2402_13533_b200 import _lib
    from paper_2402_13533_b200.decoder import DecoderConfig, build_decoder

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product has no CPU path)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    c = CONFIGS["4"]
    cfg = DecoderConfig(vocab=32000, dim=4096, heads=32, layers=DECODER_LAYERS, ffn_dim=11008, max_seq=c["seq"])
    model = build_decoder(cfg, rank=c["rank"], bits=c["bits"], seed=1, device=dev)  # same on every rank
    lib = _lib.lib()
    g = torch.Generator().manual_seed(99 + rank)  # this rank's shard of the global batch
    host_tok = torch.randint(0, cfg.vocab, (c["batch"], c["seq"]), generator=g).pin_memory()
    host_tgt = torch.randint(0, cfg.vocab, (c["batch"], c["seq"]), generator=g).pin_memory()
    host_loss = torch.empty(1, dtype=torch.float32).pin_memory()
    tokens, targets = host_tok.to(dev), host_tgt.to(dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    state = None
    for _ in range(max(args.warmup, 3)):
        _, state = model.train_step(tokens, targets, state, process_group=group)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    clk_path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else f"/tmp/qa_clocks_rank{rank}.csv"
    sampler = clocks_sampler_start(clk_path) if local == 0 else None
    time.sleep(0.4 if sampler else 0)
    n_launch0 = lib.qa_launch_count()
    lib.qa_timing_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        loss, state = model.train_step(tokens, targets, state, process_group=group)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    launches = (lib.qa_launch_count() - n_launch0) // max(args.steps, 1)
    per_class = {k: _lib.timing_read(k) for k in ("gemm_i8", "gemm_bf16", "quantize", "tt", "dequant")}
    lib.qa_timing_enable(0)
    clocks = clocks_sampler_stop(sampler, clk_path, local) if sampler else None
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    T = c["batch"] * c["seq"]
    value = T * world / (ms_step / 1e3)
    roofline, kernels = roofline_from_classes(per_class, ms_total, args.steps, clocks, with_traffic=False)

    # end to end: every step's token ids from pinned host memory, the loss read back
    e2e = None
    if not args.no_e2e:
        k_e2e = max(2, min(args.steps, 3))
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            tokens.copy_(host_tok, non_blocking=True)
            targets.copy_(host_tgt, non_blocking=True)
            loss, state = model.train_step(tokens, targets, state, process_group=group)
            host_loss.fill_(loss)
        torch.cuda.synchronize(dev)
        barrier()
        sec = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": k_e2e * T * world / sec, "unit": UNIT,
               "h2d_bytes_per_step": int(host_tok.numel() * 8 * 2), "d2h_bytes_per_step": 4, "steps": k_e2e}
    cpu = decoder_cpu_rate() if rank == 0 and world == 1 and not args.no_cpu_baseline else None
    if rank == 0:
        line = {"metric": "decoder training step tokens/s", "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int8 (u8xu8->s32) GEMM + bf16", "data": "synthetic",
                "config": decoder_desc(world), "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu,
                "e2e": e2e, "loss": loss, "gpu_launches": int(launches * args.steps),
                "gpu_launches_per_step": int(launches), "clocks": clocks,
                "note": "attention is torch SDPA (cuDNN); gpu_launches counts this library's kernels only"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- GPU arm

MERGE_70B = [("wq", 8192, 8192), ("wk", 1024, 8192), ("wv", 1024, 8192), ("wo", 8192, 8192),
             ("wu", 28672, 8192), ("wg", 28672, 8192), ("wd", 8192, 28672)]


def measure_merge(dev, sptr, hbm_gbs, iters=5):
    """qa_merge (W' = dequantize_rows(q) + W_t, lowrank.py:245-257) over the config-5 70B set, int4, r = 8; one
    matrix resident at a time.  The headline is the fp32 W' the reference's lora_merge returns (numpy float32
    dense weights, lowrank.py:254-257); the bf16 W' (the serving dtype) is reported beside it."""
    import torch

    from paper_2402_13533_b200 import _lib
    from paper_2402_13533_b200.linear import TTSpec
    from paper_2402_13533_b200.quant import quantize_rows

    lib = _lib.lib()
    res = {}
    for odt, code, tag in ((torch.float32, _lib.QA_F32, "f32"), (torch.bfloat16, _lib.QA_BF16, "bf16")):
        g = torch.Generator(device=dev).manual_seed(7)
        tot_ms, tot_bytes = 0.0, 0.0
        for name, n, k in MERGE_70B:
            w = torch.randn((n, k), generator=g, device=dev) * 0.02
            q = quantize_rows(w, 4)
            del w
            spec = TTSpec.for_shape(n, k, 8)
            cores = [torch.randn(spec.core_shape(i), generator=g, device=dev) * 0.01 for i in range(spec.d)]
            wc, ttc = q.as_c(), spec.as_c(cores)
            wsm = torch.empty(max(lib.qa_merge_workspace_bytes(ctypes.byref(ttc)), 16), dtype=torch.uint8,
                              device=dev)
            out = torch.empty((n, k), dtype=odt, device=dev)

            def run():
                _lib.check(lib.qa_merge(ctypes.byref(wc), ctypes.byref(ttc), out.data_ptr(), code, wsm.data_ptr(),
                                        wsm.numel(), sptr), "qa_merge")

            run()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                run()
            e1.record()
            torch.cuda.synchronize(dev)
            tot_ms += e0.elapsed_time(e1) / iters
            tot_bytes += n * k * 0.5 + n * k * out.element_size() + 8 * n + 4 * spec.param_count()
            del q, out, wsm, cores
        gbs = tot_bytes / tot_ms / 1e6
        res[tag] = {"ms": tot_ms, "bytes": tot_bytes, "achieved_gbs": gbs, "frac_of_hbm": gbs / hbm_gbs}
    out = {"set": "llama2-70b linears (q/o 8192^2, k/v 1024x8192, gate/up 28672x8192, down 8192x28672), int4, "
                  "TT r=8, fp32 W' (the reference's dtype)", **res["f32"], "kernels": "k_merge_fast"}
    out["bf16_out"] = res["bf16"]
    return out


def measure_weight_quantize(dev, sptr, hbm_gbs, linears, bits, iters=5):
    """qa_quantize_rows (quant.py:73-99, north-star step 1) over the config's linear set from f32 weights,
    outside the timed region: algorithmic bytes = f32 in + codes out + scale / offset / Σcodes."""
    import torch

    from paper_2402_13533_b200 import _lib

    lib = _lib.lib()
    g = torch.Generator(device=dev).manual_seed(11)
    tot_ms, tot_bytes = 0.0, 0.0
    for name, n, k, _ in linears:
        w = torch.randn((n, k), generator=g, device=dev) * 0.02
        ld = k if bits == 8 else (k + 1) // 2
        codes = torch.empty((n, ld), dtype=torch.uint8, device=dev)
        sc, of = torch.empty(n, device=dev), torch.empty(n, device=dev)
        rs = torch.empty(n, dtype=torch.int32, device=dev)

        def run():
            _lib.check(lib.qa_quantize_rows(w.data_ptr(), _lib.QA_F32, n, k, k, bits, codes.data_ptr(), ld, k,
                                            sc.data_ptr(), of.data_ptr(), rs.data_ptr(), None, sptr), "quantize")

        run()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            run()
        e1.record()
        torch.cuda.synchronize(dev)
        tot_ms += e0.elapsed_time(e1) / iters
        tot_bytes += n * k * 4 + n * ld + 12 * n
        del w, codes
    gbs = tot_bytes / tot_ms / 1e6
    return {"set": f"the config's {len(linears)} linears from f32, int{bits}", "ms": tot_ms, "bytes": tot_bytes,
            "achieved_gbs": gbs, "frac_of_hbm": gbs / hbm_gbs, "kernels": "k_quantize_rows"}


def roofline_from_classes(per_class, ms_total, steps, clocks, with_traffic=True):
    """Roofline of the dominant kernel class and every class's share / fraction of its own roofline, from the
    library's live per-launch CUDA-event durations of the timed region (qa_timing_*)."""
    # --- roofline of the dominant kernel class (live CUDA-event durations of the timed region)
    peaks, peak_src = measured_peaks()
    dom = max(per_class, key=lambda c: per_class[c][0])
    dms, dn, dwork = per_class[dom]
    kernels = {}
    for c, (cms, cn, cw) in per_class.items():
        if cn == 0:
            continue
        avg_s = cms / cn / 1e3
        if c.startswith("gemm"):
            kernels[c] = {"ms_per_step": cms / steps, "launches_per_step": cn / steps,
                          "achieved_tflops": cw / cn / avg_s / 1e12, "share_of_step": cms / ms_total}
        else:  # HBM-bound classes: work = algorithmic bytes
            kernels[c] = {"ms_per_step": cms / steps, "launches_per_step": cn / steps,
                          "achieved_gbs": cw / cn / avg_s / 1e9, "share_of_step": cms / ms_total}
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if with_traffic and os.path.exists(tfile):
        traffic = json.load(open(tfile)).get(dom)
    # Denominator: the step is ~10 ms and the clocks sampled in the timed region sit at max (no power
    # throttling), so the burst figures apply (B200_PROFILING.md: burst for a kernel timed in a short
    # window, sustained for seconds-long loops under the power cap).
    sustained = bool(clocks and clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and
                     clocks["sm_mhz"] < 0.9 * clocks["sm_max_mhz"])
    i8file = os.path.join(ROOT, "profiles", "int8_peak.json")
    i8 = json.load(open(i8file)) if os.path.exists(i8file) else {}
    if dom.startswith("gemm"):
        achieved = dwork / dn / (dms / dn / 1e3) / 1e12
        if dom == "gemm_bf16":
            peak = peaks.get("bf16_tflops_sustained" if sustained else "bf16_tflops", peaks.get("bf16_tflops"))
            note = (f"bf16 dense cuBLAS, {'sustained' if sustained else 'burst'}, of {peak_src} (MEASURED_PEAKS.json)")
        elif i8:
            peak = i8["int8_tops_sustained" if sustained else "int8_tops"]
            note = (f"int8 dense cuBLASLt (torch._int_mm), {'sustained' if sustained else 'burst'}, measured on this "
                    f"pool (profiles/int8_peak.json); NVIDIA spec 4.5 POPS")
        else:
            peak = 4500.0
            note = "int8 dense: no measured int8 peak; NVIDIA B200 spec 4.5 POPS"
        if sustained and achieved > peak:
            note += ("; frac > 1: the step interleaves memory-bound phases, so its GEMMs run above the "
                     "continuous-load (sustained) cuBLAS figure")
        roofline = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": note,
                    "work_per_launch": dwork / dn, "launch_ms": dms / dn}
    else:
        achieved = dwork / dn / (dms / dn / 1e3) / 1e9
        peak = peaks["hbm_gbs"]
        roofline = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": f"HBM copy, of {peak_src}"}

    # per-class fraction of its own roofline (same denominators as the headline roofline)
    p_bf16 = peaks.get("bf16_tflops_sustained" if sustained else "bf16_tflops", peaks.get("bf16_tflops"))
    p_i8 = i8.get("int8_tops_sustained" if sustained else "int8_tops", 4500.0) if i8 else 4500.0
    for c, kd in kernels.items():
        if c == "gemm_i8":
            kd["frac_of_peak"] = kd["achieved_tflops"] / p_i8
        elif c == "gemm_bf16":
            kd["frac_of_peak"] = kd["achieved_tflops"] / p_bf16
        else:
            kd["frac_of_peak"] = kd["achieved_gbs"] / peaks["hbm_gbs"]

    return roofline, kernels


def measure_decoder(dev, layers=32, batch=4, seq=2048, steps=3, warmup=2):
    """BASELINE config 4 on one GPU: the 32-layer Llama-2-7B-shaped decoder (vocab 32000), int8
    bases + TT r = 8 adapters on every linear and the head, PER_LAYER recompute, [4, 2048] tokens (the per-GPU
    share of the [32, 2048] global batch).  Outside the config-2 timed region; CUDA events, warm."""
    import torch

    from paper_2402_13533_b200.decoder import DecoderConfig, build_decoder

    cfg = DecoderConfig(vocab=32000, dim=4096, heads=32, layers=layers, ffn_dim=11008, max_seq=seq)
    model = build_decoder(cfg, rank=8, bits=8, seed=1, device=dev)
    g = torch.Generator(device=dev).manual_seed(2)
    tokens = torch.randint(0, cfg.vocab, (batch, seq), generator=g, device=dev)
    targets = torch.randint(0, cfg.vocab, (batch, seq), generator=g, device=dev)
    state = None
    for _ in range(warmup):
        _, state = model.train_step(tokens, targets, state)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss, state = model.train_step(tokens, targets, state)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    out = {"workload": f"llama2-7b decoder, {layers} layers + head, vocab 32000, int8 bases, TT r=8 on all linears "
                       f"and the head, PER_LAYER recompute, [{batch}, {seq}] tokens",
           "baseline_config": 4, "ms_per_step": ms, "tokens_per_s": batch * seq / (ms / 1e3), "steps": steps,
           "loss": loss, "adapter_tensors": len(state.names),
           "note": "trainer.train_step: fwd storing layer inputs + cross-entropy + bwd re-running each layer + "
                   "AdamW on the adapter cores; attention = torch SDPA"}
    del model, state
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.config == "4":
        return main_decoder(args)

    import torch
    import torch.distributed as dist

    from paper_2402_13533_b200 import _lib, dp
    from paper_2402_13533_b200.linear import QuantizedLinear, TTLinear, TTSpec
    from paper_2402_13533_b200.quant import quantize_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product has no CPU path)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, T, scaling, desc = workload_config(args.config, world)
    LINEARS, IN_DIMS = linear_set(args.config)
    lib = _lib.lib()
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    if world > 1 and rank == 0:
        print(f"[bench] {world} ranks, NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}, backend "
              f"{dist.get_backend()}", file=sys.stderr, flush=True)

    # --- frozen quantised base + TT adapters (identical on every rank: same seed)
    gen = torch.Generator(device=dev).manual_seed(1234)
    mats = {}
    ws_bytes = 0
    grad_numel = 0
    for name, n, k, kind in LINEARS:
        w = torch.randn((n, k), generator=gen, device=dev, dtype=torch.float32) * 0.02
        q = quantize_rows(w, cfg["bits"])
        del w
        spec = TTSpec.for_shape(n, k, cfg["rank"])
        cores = [torch.randn(spec.core_shape(i), generator=gen, device=dev) * 0.01 for i in range(spec.d)]
        wc, ttc = q.as_c(), spec.as_c(cores)
        ws_bytes = max(ws_bytes, lib.qa_linear_workspace_bytes(ctypes.byref(wc), ctypes.byref(ttc), T))
        nsaved = lib.qa_linear_saved_bytes(ctypes.byref(wc), ctypes.byref(ttc), T)
        saved = torch.empty(max(nsaved, 4), dtype=torch.uint8, device=dev)
        mats[name] = dict(q=q, spec=spec, cores=cores, wc=wc, ttc=ttc, n=n, k=k, kind=kind, saved=saved,
                          nsaved=nsaved)
        grad_numel += spec.param_count()
    # shared-input groups: ctypes argument arrays built once
    groups = {}
    for gnames in set(GROUPS_FWD) | set(GROUPS_BWD):
        if len(gnames) < 2:
            continue
        n = len(gnames)
        W = (ctypes.POINTER(_lib.QWeight) * n)(*[ctypes.pointer(mats[g]["wc"]) for g in gnames])
        Tt = (ctypes.POINTER(_lib.TT) * n)(*[ctypes.pointer(mats[g]["ttc"]) for g in gnames])
        ws_bytes = max(ws_bytes, lib.qa_group_workspace_bytes(n, W, Tt, T))
        groups[gnames] = dict(n=n, W=W, T=Tt)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    # one flat buffer of every adapter-core gradient (linear order, then core order): the kernels write into its
    # views and one collective averages it (dp.flat_views / dp.average_flat_, covered by tests/test_dp_gloo.py)
    flat_grad = torch.zeros(grad_numel, dtype=torch.float32, device=dev)
    grad_layout = [(f"{name}.core{i}", mats[name]["spec"].core_shape(i)) for name, _, _, _ in LINEARS
                   for i in range(mats[name]["spec"].d)]
    gviews = dp.flat_views(flat_grad, grad_layout)
    for name, n, k, kind in LINEARS:
        m = mats[name]
        m["gptr"] = (ctypes.c_void_p * _lib.QA_TT_MAX_D)(
            *[gviews[f"{name}.core{i}"].data_ptr() for i in range(m["spec"].d)])

    # every rank must hold the same frozen codes and adapter cores before the step (the state_signature check
    # of distsim.federated_round, distsim.py:293-296)
    if world > 1:
        dp.check_replicas([TTLinear(nm, QuantizedLinear(nm + ".base", mats[nm]["q"]), mats[nm]["spec"],
                                    mats[nm]["cores"]) for nm, _, _, _ in LINEARS])

    # --- per-rank synthetic activations / upstream grads (rank-dependent seed: different token shards)
    dgen = torch.Generator(device=dev).manual_seed(99 + rank)

    def make_inputs():
        xs = {kd: torch.randn((T, d), generator=dgen, device=dev).to(torch.bfloat16) for kd, d in IN_DIMS.items()}
        dys = {nm: torch.randn((T, n), generator=dgen, device=dev).to(torch.bfloat16) for nm, n, _, _ in LINEARS}
        return xs, dys

    xs, dys = make_inputs()
    ys = {nm: torch.empty((T, n), dtype=torch.bfloat16, device=dev) for nm, n, _, _ in LINEARS}
    dxs = {nm: torch.empty((T, k), dtype=torch.bfloat16, device=dev) for nm, _, k, _ in LINEARS}
    BF16 = _lib.QA_BF16

    for gnames, gd in groups.items():  # saved-state, gradient and dy/dx pointer arrays
        n = gd["n"]
        gd["S"] = (ctypes.c_void_p * n)(*[mats[g]["saved"].data_ptr() for g in gnames])
        gd["SB"] = (ctypes.c_size_t * n)(*[mats[g]["nsaved"] for g in gnames])
        gd["DC"] = (ctypes.POINTER(ctypes.c_void_p) * n)(
            *[ctypes.cast(mats[g]["gptr"], ctypes.POINTER(ctypes.c_void_p)) for g in gnames])
        gd["Y"] = (ctypes.c_void_p * n)(*[ys[g].data_ptr() for g in gnames])
        gd["DX"] = (ctypes.c_void_p * n)(*[dxs[g].data_ptr() for g in gnames])
        gd["kind"] = mats[gnames[0]]["kind"]

    def step(xs, dys):
        if not args.no_group:
            return step_grouped(xs, dys)
        for name, _, _, kind in LINEARS:
            m = mats[name]
            st = lib.qa_linear_forward_save(ctypes.byref(m["wc"]), ctypes.byref(m["ttc"]), xs[kind].data_ptr(), BF16,
                                            T, ys[name].data_ptr(), m["saved"].data_ptr(), m["nsaved"],
                                            ws.data_ptr(), ws_bytes, sptr)
            if st:
                _lib.check(st, f"forward {name}")
        for name in BACKWARD_ORDER:
            m = mats[name]
            st = lib.qa_linear_backward_saved(ctypes.byref(m["wc"]), ctypes.byref(m["ttc"]),
                                              xs[m["kind"]].data_ptr(), BF16, dys[name].data_ptr(), BF16, T,
                                              dxs[name].data_ptr(),
                                              ctypes.cast(m["gptr"], ctypes.POINTER(ctypes.c_void_p)), 0,
                                              m["saved"].data_ptr(), m["nsaved"], ws.data_ptr(), ws_bytes, sptr)
            if st:
                _lib.check(st, f"backward {name}")
        if world > 1:
            dp.average_flat_(flat_grad)

    def step_grouped(xs, dys):
        for gnames in GROUPS_FWD:
            if len(gnames) == 1:
                m = mats[gnames[0]]
                st = lib.qa_linear_forward_save(ctypes.byref(m["wc"]), ctypes.byref(m["ttc"]), xs[m["kind"]].data_ptr(),
                                                BF16, T, ys[gnames[0]].data_ptr(), m["saved"].data_ptr(), m["nsaved"],
                                                ws.data_ptr(), ws_bytes, sptr)
            else:
                gd = groups[gnames]
                st = lib.qa_group_forward(gd["n"], gd["W"], gd["T"], xs[gd["kind"]].data_ptr(), BF16, T, gd["Y"],
                                          gd["S"], gd["SB"], ws.data_ptr(), ws_bytes, sptr)
            if st:
                _lib.check(st, f"forward {gnames}")
        for gnames in GROUPS_BWD:
            if len(gnames) == 1:
                name = gnames[0]
                m = mats[name]
                st = lib.qa_linear_backward_saved(ctypes.byref(m["wc"]), ctypes.byref(m["ttc"]),
                                                  xs[m["kind"]].data_ptr(), BF16, dys[name].data_ptr(), BF16, T,
                                                  dxs[name].data_ptr(),
                                                  ctypes.cast(m["gptr"], ctypes.POINTER(ctypes.c_void_p)), 0,
                                                  m["saved"].data_ptr(), m["nsaved"], ws.data_ptr(), ws_bytes, sptr)
            else:
                gd = groups[gnames]
                DY = (ctypes.c_void_p * gd["n"])(*[dys[g].data_ptr() for g in gnames])
                st = lib.qa_group_backward(gd["n"], gd["W"], gd["T"], xs[gd["kind"]].data_ptr(), BF16, DY, BF16, T,
                                           gd["DX"], gd["DC"], 0, gd["S"], gd["SB"], ws.data_ptr(), ws_bytes, sptr)
            if st:
                _lib.check(st, f"backward {gnames}")
        if world > 1:
            dp.average_flat_(flat_grad)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # --- warm-up, then exactly K timed steps bracketed by barrier + synchronize
    for _ in range(max(args.warmup, 3)):
        step(xs, dys)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    clk_path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv") if os.path.isdir(
        os.path.join(ROOT, "gpurun_out")) else f"/tmp/qa_clocks_rank{rank}.csv"
    sampler = clocks_sampler_start(clk_path) if local == 0 else None
    time.sleep(0.4 if sampler else 0)
    n_launch0 = lib.qa_launch_count()
    lib.qa_timing_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    for _ in range(args.steps):
        step(xs, dys)
    host_issue_ms = (time.perf_counter() - h0) * 1e3 / max(args.steps, 1)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    launches = (lib.qa_launch_count() - n_launch0) // max(args.steps, 1)
    per_class = {c: _lib.timing_read(c) for c in ("gemm_i8", "gemm_bf16", "quantize", "tt", "dequant")}
    lib.qa_timing_enable(0)
    # diagnostic (outside the timed region): the same steps without the per-launch timing events
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        step(xs, dys)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    diag = {"host_issue_ms_per_step": host_issue_ms,
            "ms_per_step_without_launch_events": e2.elapsed_time(e3) / max(args.steps, 1)}
    clocks = clocks_sampler_stop(sampler, clk_path, local) if sampler else None
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = T * world / (ms_step / 1e3)

    roofline, kernels = roofline_from_classes(per_class, ms_total, args.steps, clocks)
    peaks, peak_src = measured_peaks()

    # --- end-to-end through the C ABI with host buffers: pinned H2D of every step's inputs
    # (double-buffered on a copy stream, overlapping the previous step) + D2H of the gradients
    e2e = None
    if not args.no_e2e:
        host_x = {kd: v.cpu().pin_memory() for kd, v in xs.items()}
        host_dy = {nm: v.cpu().pin_memory() for nm, v in dys.items()}
        host_grad = torch.empty(grad_numel, dtype=torch.float32).pin_memory()
        bufs = [(xs, dys), make_inputs()]
        copy_stream = torch.cuda.Stream(dev)
        h2d = sum(v.numel() * v.element_size() for v in host_x.values()) + \
            sum(v.numel() * v.element_size() for v in host_dy.values())
        d2h = host_grad.numel() * 4
        uploaded = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def upload(i):
            bx, bdy = bufs[i % 2]
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(consumed[i % 2])
                for kd in bx:
                    bx[kd].copy_(host_x[kd], non_blocking=True)
                for nm in bdy:
                    bdy[nm].copy_(host_dy[nm], non_blocking=True)
                uploaded[i % 2].record(copy_stream)

        for i in range(2):
            consumed[i].record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        k_e2e = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        upload(0)
        for i in range(k_e2e):
            if i + 1 < k_e2e:
                upload(i + 1)
            stream.wait_event(uploaded[i % 2])
            step(*bufs[i % 2])
            consumed[i % 2].record(stream)
            host_grad.copy_(flat_grad, non_blocking=True)
        torch.cuda.synchronize(dev)
        barrier()
        sec = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": k_e2e * T * world / sec, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": k_e2e,
               "note": "C-ABI calls on pinned host inputs; H2D of step i+1 overlaps compute of step i"}

    # decode-size forwards (KV-cached decoding, transformer.py:1043-1080): 1 and 8 tokens through the 7
    # linears; HBM-bound on the weight codes (gemv.cu)
    decode = None
    if rank == 0 and not args.no_merge and args.config != "5":
        decode = {}
        for td in (1, 8):
            xd = {kd: torch.randn((td, d), generator=dgen, device=dev).to(torch.bfloat16) for kd, d in IN_DIMS.items()}
            yd = {nm: torch.empty((td, n), dtype=torch.bfloat16, device=dev) for nm, n, _, _ in LINEARS}

            dgroups = {}
            for gnames in GROUPS_FWD:
                if len(gnames) > 1:
                    gd = groups[gnames]
                    dgroups[gnames] = (ctypes.c_void_p * gd["n"])(*[yd[g].data_ptr() for g in gnames])

            def dstep(sp):  # as a decoder layer calls them: q/k/v and up/gate as shared-input groups
                for gnames in GROUPS_FWD:
                    if len(gnames) == 1:
                        m = mats[gnames[0]]
                        _lib.check(lib.qa_linear_forward(ctypes.byref(m["wc"]), ctypes.byref(m["ttc"]),
                                                         xd[m["kind"]].data_ptr(), BF16, td, yd[gnames[0]].data_ptr(),
                                                         None, None, None, ws.data_ptr(), ws_bytes, sp),
                                   "decode forward")
                    else:
                        gd = groups[gnames]
                        _lib.check(lib.qa_group_forward(gd["n"], gd["W"], gd["T"], xd[gd["kind"]].data_ptr(), BF16, td,
                                                        dgroups[gnames], None, None, ws.data_ptr(), ws_bytes, sp),
                                   "decode group forward")

            def timed(fn, n=50):
                for _ in range(5):
                    fn()
                torch.cuda.synchronize(dev)
                d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                d0.record(stream)
                for _ in range(n):
                    fn()
                d1.record(stream)
                torch.cuda.synchronize(dev)
                return d0.elapsed_time(d1) / n

            ms_eager = timed(lambda: dstep(sptr))
            # the step captured once as a CUDA graph (programmatic-dependent edges included) and replayed: the
            # decode loop of a serving engine, without the host's per-call launch latency
            graph = torch.cuda.CUDAGraph()
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(stream)
            with torch.cuda.graph(graph, stream=gs):
                dstep(gs.cuda_stream)
            stream.wait_stream(gs)
            ms = timed(graph.replay)
            wbytes = sum(mats[nm]["q"].codes.numel() + 8 * n for nm, n, _, _ in LINEARS)
            decode[f"tokens_{td}"] = {"ms_per_step": ms, "tokens_per_s": td / (ms / 1e3),
                                      "weight_gbs": wbytes / ms / 1e6, "frac_of_hbm": wbytes / ms / 1e6 / peaks["hbm_gbs"],
                                      "ms_per_step_host_issued": ms_eager}
        decode["note"] = ("forward of the 7 linears for 1 / 8 tokens (int8 codes + TT adapter; q/k/v and up/gate as "
                          "shared-input groups): act-quant prologue + tensor-core matrix-vector pass per linear, chained "
                          "with programmatic dependent launches, replayed as one CUDA graph (ms_per_step_host_issued: "
                          "the same calls issued from the host each step); weight_gbs counts the code bytes read per step")

    # the merge kernel (north star step 6) on BASELINE config 5's 70B linear set (int4, TT r = 8), outside
    # the timed region: algorithmic bytes = codes in + bf16 W' out, CUDA events, warm
    merge = None
    if rank == 0 and not args.no_merge:
        merge = measure_merge(dev, sptr, peaks["hbm_gbs"])

    wquant = None
    if rank == 0 and not args.no_merge:
        wquant = measure_weight_quantize(dev, sptr, peaks["hbm_gbs"], LINEARS, cfg["bits"])

    decoder = None
    if rank == 0 and world == 1 and not args.no_decoder and args.config != "5":
        decoder = measure_decoder(dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(args.config, 64 if args.config == "5" else 1024)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "int8 (u8xu8->s32) GEMM + bf16", "data": "synthetic",
            "config": desc, "roofline": roofline, "kernels": kernels, "decode": decode, "merge": merge,
            "weight_quantize": wquant, "decoder": decoder,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches * args.steps), "gpu_launches_per_step": int(launches), "clocks": clocks,
            "diagnostics": diag,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
