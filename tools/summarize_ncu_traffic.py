"""Per-kernel time + DRAM traffic from an ncu CSV (metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum) of one forward; writes JSON summary."""
import csv, sys, json, collections
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr = r; start = i + 1; break
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
for r in rows[start:]:
    if len(r) <= vi: continue
    try: v = float(r[vi].replace(",", ""))
    except ValueError: continue
    per[r[idi]][r[mi]] = v * scale.get(r[ui], 1)
    names[r[idi]] = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("pearl::", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k, m in per.items():
    a = agg[names[k]]
    a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0); a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
T = sum(a[1] for a in agg.values()); B = sum(a[2] for a in agg.values())
out = {"kernels": {n: {"launches": a[0], "time_us": round(a[1] * 1e6, 1), "share": round(a[1] / T, 4),
                       "dram_bytes": int(a[2]), "GBps": round(a[2] / a[1] / 1e9, 1) if a[1] else None}
                   for n, a in sorted(agg.items(), key=lambda x: -x[1][1])},
       "total_time_us": round(T * 1e6, 1), "total_dram_bytes": int(B), "launches": sum(a[0] for a in agg.values())}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
