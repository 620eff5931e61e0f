"""Summarise an ncu --metrics gpu__time_duration.sum CSV into per-kernel totals."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr = r; start = i + 1; break
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[start:]:
    if len(r) <= vi: continue
    try: v = float(r[vi].replace(",", ""))
    except ValueError: continue
    k = r[ki].split("(")[0]
    tot[k] += v; cnt[k] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:45s} n={cnt[k]:5d} total={v/1e3:9.1f} us  share={100*v/T:5.1f}%  avg={v/cnt[k]/1e3:8.2f} us")
print(f"TOTAL {T/1e3:.1f} us over {sum(cnt.values())} launches")
