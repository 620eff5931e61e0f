"""Single-token forward time of each draft model on both GEMM engines
(CUDA-core GEMV K2 vs tcgen05 K3), with achieved weight-streaming GB/s."""
import sys, os, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import llama
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["llama-68m", "dsc-1.3b", "llama3-8b"]
for name in names:
    cfg = llama.PRESETS[name]
    align = llama.AlignSpec()
    shared = llama._shared_tables(cfg.vocab, align, "cuda")
    w = llama.init_weights(cfg, align, 3, "cuda", shared)
    del shared
    for kind in ("cudacore", "tcgen05"):
        m = llama.LlamaModel(cfg, w, gemm=kind, max_seq=256, max_tokens=64)
        for M in (1, 4):
            t = m.measure_forward_time(M, iters=10)
            print(f"{name:10s} {kind:8s} M={M}: {t*1e3:7.3f} ms  {cfg.weight_bytes()/t/1e9:7.0f} GB/s", flush=True)
        m.close(); del m
    del w; gc.collect(); torch.cuda.empty_cache()
