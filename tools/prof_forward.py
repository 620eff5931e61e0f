"""Target window forwards of a named model (for ncu launch lists / full captures).

    python tools/prof_forward.py llama2-7b 4 [tcgen05|cudacore] [iters]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import llama

name = sys.argv[1]
M = int(sys.argv[2])
gemm = sys.argv[3] if len(sys.argv) > 3 else "tcgen05"
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
flags = int(os.environ.get("FWD_FLAGS", "0"))  # 4 = PEARL_FWD_PERSISTENT
cfg = llama.PRESETS[name]
align = llama.AlignSpec()
shared = llama._shared_tables(cfg.vocab, align, "cuda")
w = llama.init_weights(cfg, align, 7, "cuda", shared)
m = llama.LlamaModel(cfg, w, gemm=gemm, max_seq=512, max_tokens=64)
toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
pos = torch.tensor([192], dtype=torch.int32, device="cuda")
out = torch.empty(M, cfg.vocab, device="cuda")
def timed(stream, graph=False):
    with torch.cuda.stream(stream):
        for _ in range(iters):
            m.forward(toks, M, pos, flags, out, stream)
        g = None
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                m.forward(toks, M, pos, flags, out)
        stream.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(5):
            if g is not None:
                g.replay()
            else:
                m.forward(toks, M, pos, flags, out, stream)
        e.record(); e.synchronize()
        return s.elapsed_time(e) / 5
for label, st, gr in (("default-stream", torch.cuda.default_stream(), False), ("side-stream", torch.cuda.Stream(), False),
                      ("cuda-graph", torch.cuda.Stream(), True)):
    t = timed(st, gr)
    print(f"{name} M={M} {gemm} {label}: {t:.3f} ms/forward, {cfg.weight_bytes()/(t/1e3)/1e9:.0f} GB/s weights", flush=True)

import numpy as np, ctypes
from paper_2408_11850_b200 import _lib
names = ["embed", "norm", "qkv", "attn", "o", "gate_up", "down", "lm_head", "other", "TOTAL"]
buf = (ctypes.c_float * 10)()
for rep in range(3):
    _lib.load().pearl_llama_profile(m.handle, toks.data_ptr(), M, pos.data_ptr(), out.data_ptr(), buf,
                                    torch.cuda.current_stream().cuda_stream)
print("per-op ms (events between launches):", {n: round(buf[i], 3) for i, n in enumerate(names)})

# persistent-kernel phase timeline (tcgen05 models, M <= 16)
if gemm == "tcgen05" and M <= 16:
    kinds = {0: "embed", 1: "norm", 2: "gemm", 3: "attn"}
    tr = (ctypes.c_float * (3 * 2000))()
    for rep in range(2):
        n = _lib.load().pearl_llama_mega_trace(m.handle, toks.data_ptr(), M, pos.data_ptr(), 0, out.data_ptr(), tr,
                                               2000, torch.cuda.current_stream().cuda_stream)
    assert n > 0, _lib.load().pearl_last_error()
    per = {}
    prev = 0.0
    rows = []
    for p in range(n):
        k, hi, lo = kinds[int(tr[3 * p])], tr[3 * p + 1], tr[3 * p + 2]
        per.setdefault(k, [0.0, 0])
        per[k][0] += hi - prev
        per[k][1] += 1
        rows.append((p, k, round(hi - prev, 2), round(hi - lo, 2)))
        prev = hi
    print(f"mega trace: total {prev:.1f} us over {n} phases;",
          {k: (round(v[0], 1), v[1]) for k, v in per.items()}, flush=True)
    print("first layer phases (p, kind, us since prev end, spread last-first):", rows[:9], flush=True)
    print("last phases:", rows[-4:], flush=True)
