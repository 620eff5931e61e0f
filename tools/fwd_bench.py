"""Graph-replayed forward time of one model at several window sizes M and
context positions (CUDA events, back-to-back replays), with the roofline
fraction of its algorithmic bytes.

    python tools/fwd_bench.py [preset] [gemm] [M,M,..] [ctx,ctx,..]
    PEARL_ABLATE=attn python tools/fwd_bench.py ...   # attention skipped
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_11850_b200 import llama  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
gemm = sys.argv[2] if len(sys.argv) > 2 else "tcgen05"
Ms = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,4,8,16,32").split(",")]
ctxs = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "192,500").split(",")]
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6449.7
cfg = llama.PRESETS[name]
align = llama.AlignSpec()
w = llama.init_weights(cfg, align, 7, "cuda", llama._shared_tables(cfg.vocab, align, "cuda"))
m = llama.LlamaModel(cfg, w, gemm=gemm, max_seq=1024, max_tokens=128 if gemm == "tcgen05" else 64)
res = {}
for ctx in ctxs:
    for M in Ms:
        toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
        pos = torch.tensor([ctx], dtype=torch.int32, device="cuda")
        out = torch.empty(M, cfg.vocab, device="cuda")
        for _ in range(3):
            m.forward(toks, M, pos, 0, out)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            m.forward(toks, M, pos, 0, out)
        for _ in range(3):
            g.replay()
        n = 20
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            g.replay()
        e.record()
        e.synchronize()
        t = s.elapsed_time(e) / 1e3 / n
        byts = cfg.weight_bytes() + cfg.kv_bytes_per_token() * (ctx + M) + 4 * M * cfg.vocab
        res[f"M{M}_ctx{ctx}"] = {"ms": round(t * 1e3, 4), "GBps": round(byts / t / 1e9, 1),
                                 "frac": round(byts / t / 1e9 / peak, 4)}
        print(name, gemm, f"M={M} ctx={ctx}", res[f"M{M}_ctx{ctx}"], os.environ.get("PEARL_ABLATE", ""), flush=True)
        del g
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/fwd_bench_{name}_{gemm}{'_abl' + os.environ['PEARL_ABLATE'] if 'PEARL_ABLATE' in os.environ else ''}.json", "w") as fh:
    json.dump(res, fh, indent=1)
