"""Print the last N launches of an ncu --csv launch list: python tools/lastlaunch.py file.csv N"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[i]
ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d = OrderedDict()
for r in rows[i + 1:]:
    if len(r) > vi:
        d.setdefault((r[idi], r[ki].split("(")[0][-40:]), {})[r[mi]] = r[vi]
for (id_, k), m in list(d.items())[-int(sys.argv[2]):]:
    print(id_, k, " ".join(f"{kk.split('.')[0].split('__')[-1]}={v}" for kk, v in m.items()))
