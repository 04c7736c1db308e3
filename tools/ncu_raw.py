"""Key metrics of an `ncu --page raw --csv` export, one block per profiled kernel (stall reasons above 0.1 only).
    python tools/ncu_raw.py raw.csv [regex-of-extra-metrics]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
pat = (r"gpu__time_duration.sum|dram__bytes_(read|write).sum$|smsp__inst_executed.sum$|issue_active.avg.pct"
       r"|warps_active.avg.pct|registers_per_thread$|dram_throughput.avg.pct_of_peak_sustained_elapsed|grid_size"
       r"|stalled_.*_per_issue_active|lts__t_sector_hit_rate.pct|occupancy_limit_(registers|shared_mem)")
if len(sys.argv) > 2:
    pat += "|" + sys.argv[2]
ik = hdr.index("Kernel Name")
for r in rows[2:]:
    print(r[ik][:90])
    for i, h in enumerate(hdr):
        if re.search(pat, h):
            try:
                if "stalled" in h and float(r[i]) < 0.1:
                    continue
            except ValueError:
                pass
            print("   ", h, r[i])
