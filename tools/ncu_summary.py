"""Summarise an ncu report (or a launch-list CSV) into the plain-text files kept under profiles/.

    python tools/ncu_summary.py report.ncu-rep > profiles/rNN_ncu_<what>.txt
    python tools/ncu_summary.py --launches launches.csv [LAST_N] > profiles/rNN_launch_list_summary.txt
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "IMMA subpipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "HMMA subpipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def summarise_report(path: str) -> str:
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` output saved on the GPU box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"ncu report: {path}"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        out.append(f"\n== {name}")
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"  {label:28s} {r[i]} {units[i]}")
    return "\n".join(out) + "\n"


def summarise_launches(path: str, last: int = 0) -> str:
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if "Kernel Name" in l)
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    if "Metric Name" in hdr:  # keep the duration rows only (the list may carry other metrics)
        mi = hdr.index("Metric Name")
        rows = [hdr] + [r for r in rows[1:] if len(r) > mi and r[mi] == "gpu__time_duration.sum"]
    if last:
        rows = [hdr] + [r for r in rows[1:] if len(r) > 1][-last:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        v = float(r[vi].replace(",", "")) * scale
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
    out = [f"launch list: {path} (cold-cache, serialised under ncu: compare shares, not absolutes)",
           f"{'us':>10s} {'n':>4s} {'share':>6s}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{t:10.1f} {n:4d} {100 * t / total:5.1f}%  {k}")
    out.append(f"total {total:.1f} us over {sum(a[0] for a in agg.values())} launches")
    return "\n".join(out) + "\n"


def per_launch(path: str, last: int) -> str:
    """Duration, DRAM read / write and rate of each of the last `last` launches of a launch-list CSV taken with
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum."""
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if "Kernel Name" in l)
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ii, ki, mi = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name")
    vi, ui = hdr.index("Metric Value"), hdr.index("Metric Unit")
    launches = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki].split("(")[0]})
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1e-6,
                 "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(r[ui], 1.0)
        d[r[mi]] = float(r[vi].replace(",", "")) * scale
    out = ["per launch, one timed step (cold cache, serialised): duration, DRAM read / write, DRAM rate"]
    for d in list(launches.values())[-last:]:
        us = d.get("gpu__time_duration.sum", 0.0)
        rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        rate = (rd + wr) / us if us else 0.0  # MB / us = TB/s
        out.append(f"{us:8.1f} us  rd {rd:9.1f} MB  wr {wr:8.1f} MB  {rate:5.2f} TB/s  {d['name']}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        sys.stdout.write(summarise_launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0))
    elif sys.argv[1] == "--per-launch":
        sys.stdout.write(per_launch(sys.argv[2], int(sys.argv[3])))
    else:
        sys.stdout.write(summarise_report(sys.argv[1]))
