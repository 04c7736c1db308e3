"""Per-kernel hot spots of an `ncu --page source --csv` (SASS) export holding several kernels:
    python tools/src_stalls.py src.csv SECTION [stall_column] [top]   (SECTION = 0, 1, ... in file order)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
sec = int(sys.argv[2])
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = hdrs[sec]
end = hdrs[sec + 1] - 1 if sec + 1 < len(hdrs) else len(rows)
hdr = rows[h]
ic, isrc, iex = hdr.index(col), hdr.index("Source"), hdr.index("Instructions Executed")
data = []
for r in rows[h + 1:end]:
    if len(r) <= ic:
        continue
    try:
        data.append((int(float(r[ic] or 0)), int(float(r[iex] or 0)), r[0], r[isrc].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print(f"section {sec}: {len(data)} instructions, {col} total {tot}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:7d} {d[1]:9d} {d[2][-5:]} {d[3][:90]}")
