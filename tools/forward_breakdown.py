"""Per-kernel breakdown of the LAST forward in an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv):
kernels from the last embed_kernel on, grouped by name, with time share and GB/s.

    python tools/forward_breakdown.py gpurun_out/launches_7b_m4_r02.csv [--json out.json]
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr, start = r, i + 1
        break
ID, KN, MN, MV = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
launch = collections.OrderedDict()
for r in rows[start:]:
    if len(r) <= MV:
        continue
    d = launch.setdefault(r[ID], {"name": r[KN].split("(")[0].replace("void ", "")})
    try:
        d[r[MN]] = float(r[MV].replace(",", ""))
    except ValueError:
        pass
L = list(launch.values())
last = max(i for i, d in enumerate(L) if "embed_kernel" in d["name"])
fw = [d for d in L[last:] if "pearl" in d["name"]]
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in fw:
    t = tot[d["name"]]
    t[0] += 1
    t[1] += d.get("gpu__time_duration.sum", 0)
    t[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
T = sum(v[1] for v in tot.values())
B = sum(v[2] for v in tot.values())
out = {}
for k, (n, t, b) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    out[k] = {"launches": n, "us": round(t / 1e3, 1), "share": round(t / T, 4), "dram_MB": round(b / 1e6, 1),
              "GBps": round(b / t, 1) if t else None}
    print(f"{k:40s} n={n:4d} {t/1e3:9.1f} us {100*t/T:5.1f}%  {b/1e6:9.1f} MB  {b/t if t else 0:7.1f} GB/s")
print(f"TOTAL {T/1e3:.1f} us, {B/1e9:.3f} GB, {len(fw)} launches")
if "--json" in sys.argv:
    json.dump({"kernels": out, "total_us": round(T / 1e3, 1), "total_GB": round(B / 1e9, 4), "launches": len(fw)},
              open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
