"""Print the last N launches (kernel, us, DRAM MB, grid) of an ncu --metrics CSV."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 13
hdr = rows[0]
ki, mi, vi, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = defaultdict(dict)
for r in rows[1:]:
    d[int(r[idi])][r[mi]] = r[vi]
    d[int(r[idi])]["k"] = r[ki].split("(")[0][-36:]
tot = 0.0
for i in sorted(d)[-n:]:
    x = d[i]
    t = float(x["gpu__time_duration.sum"]) / 1e3
    tot += t
    print(f"{x['k']:38s} {t:7.2f} us {float(x['dram__bytes_read.sum'])/1e6:7.2f} MB grid {x['launch__grid_size']}")
print(f"total {tot:.1f} us")
