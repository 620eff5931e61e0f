"""A/B of the tcgen05 GEMM's weight layout: row-major [N, K] vs tile-major
[N/128][K/64][128][64] (PEARL_GEMM_W_TILED).  The 7B layer's four GEMMs
back to back over 8 distinct layers (3.2 GB of weights: HBM-resident), in a
CUDA graph; GB/s of weights.

    python tools/gemm_layout_probe.py [M,M,..] [preset]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import _lib, llama

Ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,4,16").split(",")]
cfg = llama.PRESETS[sys.argv[2] if len(sys.argv) > 2 else "llama2-7b"]
d, F, hd = cfg.d_model, cfg.ffn, cfg.head_dim
shapes = [((cfg.n_heads + 2 * cfg.n_kv_heads) * hd, d), (d, cfg.n_heads * hd), (2 * F, d), (d, F)]
NL = 8
lib = _lib.load()


def tile(W):
    N, K = W.shape
    return W.view(N // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous()


Ws = [[(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for (N, K) in shapes] for _ in range(NL)]
Wt = [[tile(W) for W in layer] for layer in Ws]
nbytes = sum(N * K * 2 for N, K in shapes) * NL
res = {}
for M in Ms:
    X = torch.randn(M, max(K for _, K in shapes), device="cuda").to(torch.bfloat16)
    Y = torch.empty(M, max(N for N, _ in shapes), device="cuda")
    for name, WW, kind in (("rowmajor", Ws, 1), ("tiled", Wt, 1 | 0x100)):
        def run():
            st = torch.cuda.current_stream().cuda_stream
            for layer in WW:
                for W, (N, K) in zip(layer, shapes):
                    rc = lib.pearl_gemm(kind, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, 0, st)
                    assert rc == 0, rc
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        for _ in range(3):
            g.replay()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10):
            g.replay()
        e.record()
        e.synchronize()
        t = s.elapsed_time(e) / 1e3 / 10
        res[f"M{M}_{name}"] = {"us_per_layer": round(t / NL * 1e6, 2), "GBps": round(nbytes / t / 1e9, 1)}
        print(M, name, res[f"M{M}_{name}"], flush=True)
    # correctness: tiled == rowmajor bitwise
    Y1 = torch.empty(M, shapes[2][0], device="cuda")
    Y2 = torch.empty_like(Y1)
    lib.pearl_gemm(1, Ws[0][2].data_ptr(), X.data_ptr(), Y1.data_ptr(), M, *shapes[2], 0, 0)
    lib.pearl_gemm(1 | 0x100, Wt[0][2].data_ptr(), X.data_ptr(), Y2.data_ptr(), M, *shapes[2], 0, 0)
    torch.cuda.synchronize()
    print("bitwise equal:", torch.equal(Y1, Y2), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/gemm_layout_probe.json", "w"), indent=1)
