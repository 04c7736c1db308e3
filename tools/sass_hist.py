"""Histogram of an `ncu --page source --csv` (SASS view) export: instructions executed and stall
samples per opcode, plus the hottest instructions.   python tools/sass_hist.py src.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
ia, isrc, iss, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
ops = collections.Counter()
stalls = collections.Counter()
lines = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    s = r[isrc].strip()
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    try:
        n = float(r[iex] or 0)
        st = float(r[iss] or 0)
    except ValueError:  # a repeated header (several kernels in one export)
        continue
    ops[op] += n
    stalls[op] += st
    lines.append((n, st, r[ia][-5:], s[:90]))
tot = sum(ops.values())
print(f"total warp instructions {tot:.0f}, stall samples {sum(stalls.values()):.0f}")
for op, n in ops.most_common(top):
    print(f"{op:12s} {n:12.0f} {100 * n / tot:5.1f}%  stalls {stalls[op]:8.0f}")
print("-- hottest by stall samples")
for n, st, a, s in sorted(lines, key=lambda t: -t[1])[:top]:
    print(f"{n:10.0f} {st:6.0f} {a} {s}")
