"""Per-CTA timeline of a graph-replayed target forward (diagnostic build).

    python -m paper_2408_11850_b200.build --timeline     # build/var_tl/libpearl_tl.so
    PEARL_LIB_PATH=build/var_tl/libpearl_tl.so python tools/timeline.py [preset] [M] [ctx]

Stamps (globaltimer ns, per CTA): GEMM 0 entry, 1 producer past the PDL
wait, 2 first MMA, 3 last MMA commit, 4 exit; attention 0 entry, 1 past the
wait, 4 exit.  Prints, per launch: start / end (first entry, last exit)
relative to the forward's start, the spread of the PDL-wait release, the
MMA span, and the gap to the previous launch's last exit.
"""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_11850_b200 import _lib, llama  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 192
lib = _lib.load()
lib.pearl_tl_enable.argtypes = [ctypes.c_int]
lib.pearl_tl_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = llama.PRESETS[name]
align = llama.AlignSpec()
w = llama.init_weights(cfg, align, 7, "cuda", llama._shared_tables(cfg.vocab, align, "cuda"))
m = llama.LlamaModel(cfg, w, gemm="tcgen05", max_seq=max(1024, ctx + 2 * M), max_tokens=128)
toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
pos = torch.tensor([ctx], dtype=torch.int32, device="cuda")
out = torch.empty(M, cfg.vocab, device="cuda")
for _ in range(2):
    m.forward(toks, M, pos, 0, out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
NL = 8 * cfg.n_layers + 8
lib.pearl_tl_enable(NL)
with torch.cuda.graph(g):
    m.forward(toks, M, pos, 0, out)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
buf = np.zeros((NL, 160, 16), dtype=np.uint64)
n = lib.pearl_tl_read(buf.ctypes.data, NL)
buf = buf[:n].astype(np.int64)
kinds = []
per_layer = 5  # qkv, attn, o, gate_up, down
for i in range(n):
    if i == n - 1:
        kinds.append("lm_head")
    else:
        kinds.append(["qkv", "attn", "o", "gate_up", "down"][i % per_layer])
t0 = min(int(b[:, 0][b[:, 0] > 0].min()) for b in buf[:1])
rows = []
prev_end = None
for i in range(n):
    b = buf[i]
    live = b[:, 0] > 0
    st = b[live]
    start, end = int(st[:, 0].min()), int(st[:, 4].max())
    rel = lambda x: (x - t0) / 1e3  # noqa: E731
    r = {"i": i, "kind": kinds[i], "ctas": int(live.sum()), "start_us": round(rel(start), 2), "end_us": round(rel(end), 2),
         "dur_us": round((end - start) / 1e3, 2)}
    if kinds[i] == "attn":
        w1 = st[:, 1][st[:, 1] > 0]
        if len(w1):
            r.update(wait_lo=round(rel(int(w1.min())), 2), wait_hi=round(rel(int(w1.max())), 2),
                     exit_lo=round(rel(int(st[:, 4].min())), 2))
            # per-phase medians over CTAs: wait -> warp passes -> CTA fold -> cluster sync -> fold out -> exit
            ok = (st[:, 1] > 0) & (st[:, 2] > 0) & (st[:, 3] > 0) & (st[:, 5] > 0) & (st[:, 6] > 0)
            if ok.any():
                q = st[ok]
                med = lambda a, b: round(float(np.median(q[:, b] - q[:, a])) / 1e3, 2)  # noqa: E731
                r.update(ph_pass=med(1, 2), ph_ctafold=med(2, 3), ph_csync=med(3, 5), ph_foldout=med(5, 6),
                         ph_exit=med(6, 4))
    if kinds[i] != "attn":
        w1 = st[:, 1][st[:, 1] > 0]
        m2, m3 = st[:, 2][st[:, 2] > 0], st[:, 3][st[:, 3] > 0]
        r.update(wait_lo=round(rel(int(w1.min())), 2), wait_hi=round(rel(int(w1.max())), 2),
                 mma_first=round(rel(int(m2.min())), 2), mma_last_lo=round(rel(int(m3.min())), 2),
                 mma_last_hi=round(rel(int(m3.max())), 2), exit_lo=round(rel(int(st[:, 4].min())), 2))
    if prev_end is not None:
        r["gap_from_prev_end_us"] = round((start - prev_end) / 1e3, 2)
    prev_end = end
    rows.append(r)
tot = (int(buf[n - 1][:, 4].max()) - t0) / 1e3
print(f"{name} M={M} ctx={ctx}: {n} launches, forward {tot:.1f} us (first entry -> last exit)")
agg = {}
for r in rows:
    a = agg.setdefault(r["kind"], {"n": 0, "dur": 0.0, "tail": 0.0, "head": 0.0})
    a["n"] += 1
    a["dur"] += r["dur_us"]
    if "mma_last_hi" in r:
        a["tail"] += r["end_us"] - r["mma_last_hi"]   # epilogue / reduction after the last MMA
        a["head"] += r["mma_first"] - r["start_us"]   # entry -> first MMA
for k, a in agg.items():
    print(f"  {k:8s} n={a['n']:3d} dur {a['dur']/a['n']:7.2f} us  head {a['head']/a['n']:6.2f}  tail {a['tail']/a['n']:6.2f}")
for r in rows[5:10] + rows[-2:]:
    print("  ", r)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open(f"gpurun_out/timeline_{name}_M{M}.json", "w"), indent=1)

# latest-finishing CTAs of layer 1's GEMMs: last MMA (3), last accumulator seen by the
# epilogue (5), last reduction start (6), exit (4)
for i in (5, 7, 8, 9):
    b = buf[i]
    live = b[:, 0] > 0
    if not live.any() or kinds[i] == "attn":
        continue
    st_ = b[live]
    idx = np.argsort(-st_[:, 4])[:4]
    rel = lambda x: round((int(x) - t0) / 1e3, 2) if x > 0 else None  # noqa: E731
    print(f"  {kinds[i]:8s} latest: " + "; ".join(
        f"mma_end {rel(st_[j, 3])} acc {rel(st_[j, 5])} reduce {rel(st_[j, 6])} fence {rel(st_[j, 9])} "
        f"staged {rel(st_[j, 7])} epi {rel(st_[j, 8])} exit {rel(st_[j, 4])}" for j in idx))
