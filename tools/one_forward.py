"""One target window forward (for ncu launch lists / captures).

    python tools/one_forward.py llama2-7b 4 [ctx] [reps]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import llama
name, M = sys.argv[1], int(sys.argv[2])
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 192
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = llama.PRESETS[name]
align = llama.AlignSpec()
w = llama.init_weights(cfg, align, 7, "cuda", llama._shared_tables(cfg.vocab, align, "cuda"))
m = llama.LlamaModel(cfg, w, gemm="tcgen05", max_seq=1024, max_tokens=128)
toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
pos = torch.tensor([ctx], dtype=torch.int32, device="cuda")
out = torch.empty(M, cfg.vocab, device="cuda")
for _ in range(2):
    m.forward(toks, M, pos, 0, out)
torch.cuda.synchronize()
for _ in range(reps):
    m.forward(toks, M, pos, 0, out)
torch.cuda.synchronize()
print("done")
