"""Per-op device time from an ncu launch list of ONE eager forward (ops in
forward_chunk order: embed, per layer [norm, qkv, attn, o, norm, gate_up,
down], final norm, lm_head)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n_layers = int(sys.argv[2]) if len(sys.argv) > 2 else 32
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr = r; start = i + 1; break
ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
seq = []
for r in rows[start:]:
    if len(r) <= vi: continue
    try: v = float(r[vi].replace(",", ""))
    except ValueError: continue
    seq.append((r[ki].split("(")[0], v))
names = ["embed"] + ["norm1", "qkv", "attn", "o", "norm2", "gate_up", "down"] * n_layers + ["normf", "lm_head"]
tot = collections.defaultdict(float)
for (k, v), n in zip(seq, names):
    tot[n] += v
T = sum(tot.values())
print({n: round(v / 1e3, 1) for n, v in tot.items()}, "total us:", round(T / 1e3, 1))
print("per-layer avg us:", {n: round(tot[n] / 1e3 / n_layers, 2) for n in ["norm1", "qkv", "attn", "o", "norm2", "gate_up", "down"]})
