"""bench.py's measurement contract on CPU: the reference arm (the oracle port timed on the host, no GPU
involved) prints one JSON line with the keys the driver reads, for the linear set (config 2) and the
decoder stack (config 4); the roofline helper turns the library's per-class timings into fractions of the
measured peaks."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_linear_set():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    # lrlm itself when baseline/_ref holds it, else the oracle port
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["baseline_config"] == 2


def test_reference_arm_decoder_config():
    d = _run("--impl", "reference", "--config", "4", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["config"]["baseline_config"] == 4 and d["scaling"] == "weak"


def test_roofline_from_classes():
    sys.path.insert(0, ROOT)
    import bench

    # ms, launches, work (flops for GEMMs, bytes for the streaming classes) over 2 steps
    per_class = {"gemm_i8": (4.0, 14, 14 * 6.0e11), "gemm_bf16": (8.0, 14, 14 * 1.0e12), "quantize": (1.0, 8, 8 * 2e8),
                 "tt": (2.0, 64, 64 * 5e7), "dequant": (0.4, 14, 14 * 5e7)}
    roof, kernels = bench.roofline_from_classes(per_class, 18.0, 2, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0})
    assert roof["kernel"] == "gemm_bf16" and roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s"
    assert abs(roof["achieved"] - 1.0e12 / (8.0 / 14 / 1e3) / 1e12) < 1e-6
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-12
    assert set(kernels) == set(per_class)
    assert abs(sum(k["share_of_step"] for k in kernels.values()) - 15.4 / 18.0) < 1e-9
    for k in kernels.values():
        assert k["frac_of_peak"] > 0
