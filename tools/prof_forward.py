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
cfg = llama.PRESETS[name]
align = llama.AlignSpec()
shared = llama._shared_tables(cfg.vocab, align, "cuda")
w = llama.init_weights(cfg, align, 7, "cuda", shared)
m = llama.LlamaModel(cfg, w, gemm=gemm, max_seq=512, max_tokens=64)
toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
pos = torch.tensor([192], dtype=torch.int32, device="cuda")
out = torch.empty(M, cfg.vocab, device="cuda")
for _ in range(iters):
    m.forward(toks, M, pos, 0, out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(5):
    m.forward(toks, M, pos, 0, out)
e.record(); e.synchronize()
print(f"{name} M={M} {gemm}: {s.elapsed_time(e)/5:.3f} ms/forward, {cfg.weight_bytes()/(s.elapsed_time(e)/5e3)/1e9:.0f} GB/s weights")
