"""DRAM bytes (read + write) and time of the LAST target forward in an ncu
--metrics CSV of tools/one_forward.py (2 warm-up forwards + 1; a forward =
the launches from its embedding kernel on)."""
import csv, json, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
per, names = defaultdict(dict), {}
for r in rows[1:]:
    per[int(r[idi])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    names[int(r[idi])] = r[ki]
ids = sorted(per)
starts = [i for i in ids if "embed_kernel" in names[i]]
last = [i for i in ids if i >= starts[-1]]
byts = sum(per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0) for i in last)
t = sum(per[i].get("gpu__time_duration.sum", 0) for i in last)
print(json.dumps({"launches": len(last), "dram_bytes": int(byts), "time_us_serialised": round(t * 1e6, 1)}))
