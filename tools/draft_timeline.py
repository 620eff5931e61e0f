"""Phase timeline of the persistent single-token draft forward (diagnostic build).

    python -m paper_2408_11850_b200.build --timeline
    PEARL_LIB_PATH=build/var_tl/libpearl_tl.so python tools/draft_timeline.py [preset] [ctx]

Stamps per CTA: 0 entry, 1 past the PDL wait, 2.. after each grid barrier,
15 exit.  Prints the phase boundaries (median over CTAs, us from entry).
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_11850_b200 import _lib, llama  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama-68m"
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 192
lib = _lib.load()
lib.pearl_tl_enable.argtypes = [ctypes.c_int]
lib.pearl_tl_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = llama.PRESETS[name]
align = llama.AlignSpec()
w = llama.init_weights(cfg, align, 7, "cuda", llama._shared_tables(cfg.vocab, align, "cuda"))
m = llama.LlamaModel(cfg, w, gemm="cudacore", max_seq=1024, max_tokens=64)
tok = torch.full((1,), 5, dtype=torch.int32, device="cuda")
pos = torch.tensor([ctx], dtype=torch.int32, device="cuda")
out = torch.empty(1, cfg.vocab, device="cuda")
for _ in range(3):
    m.forward(tok, 1, pos, 0, out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(4):
        m.forward(tok, 1, pos, 0, out)
g.replay()
torch.cuda.synchronize()
lib.pearl_tl_enable(64)
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    for _ in range(4):
        m.forward(tok, 1, pos, 0, out)
for _ in range(2):
    g2.replay()
torch.cuda.synchronize()
buf = np.zeros((64, 160, 16), dtype=np.uint64)
n = lib.pearl_tl_read(buf.ctypes.data, 64)
print(f"{name} ctx={ctx}: {n} launches captured")
labels = ["pdl_wait"] + [f"{ph}{l}" for l in range(cfg.n_layers) for ph in ("qkv", "attn", "o", "gu", "down")][:12]
for i in range(min(n, 4)):
    b = buf[i].astype(np.int64)
    live = b[:, 0] > 0
    st = b[live]
    t0 = int(np.median(st[:, 0]))
    marks = [int(np.median(st[:, k][st[:, k] > 0])) - t0 if (st[:, k] > 0).any() else None for k in range(1, 14)]
    end = int(np.median(st[:, 15][st[:, 15] > 0])) - t0
    prev = 0
    parts = []
    for lab, mk in zip(labels, marks):
        if mk is None:
            continue
        parts.append(f"{lab}:{(mk - prev) / 1e3:.1f}")
        prev = mk
    parts.append(f"head:{(end - prev) / 1e3:.1f}")
    spread = (int(st[:, 0].max()) - int(st[:, 0].min())) / 1e3
    print(f"  launch {i}: total {end / 1e3:.1f} us (entry spread {spread:.1f}) | " + " ".join(parts))
