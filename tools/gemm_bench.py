"""Microbenchmark of the contraction engines on the decode shapes (GB/s of weights)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import _lib

SHAPES = {"7b.qkv": (12288, 4096), "7b.o": (4096, 4096), "7b.gate_up": (22016, 4096), "7b.down": (4096, 11008),
          "7b.lm_head": (32000, 4096), "68m.qkv": (2304, 768), "68m.gate_up": (6144, 768), "68m.down": (768, 3072),
          "68m.lm_head": (32000, 768)}
lib = _lib.load()
out = {}
for name, (N, K) in SHAPES.items():
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for M in (1, 4, 8, 16, 32):
        X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Y = torch.empty(M, N, device="cuda")
        for kind in (0, 1):
            st = torch.cuda.current_stream().cuda_stream
            f = lambda: lib.pearl_gemm(kind, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, 0, st)
            for _ in range(3):
                f()
            ts = []
            for _ in range(10):
                flush.zero_()
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record(); f(); e.record(); e.synchronize()
                ts.append(s.elapsed_time(e) / 1e3)
            t = sorted(ts)[len(ts) // 2]
            gbs = (N * K * 2) / t / 1e9
            out[f"{name}.M{M}.{'tc' if kind else 'gemv'}"] = round(gbs, 1)
    print(name, "splits", lib.pearl_gemm_splits(N, K), {k.split('.', 2)[2]: v for k, v in out.items() if k.startswith(name)}, flush=True)
json.dump(out, open(os.path.join(os.environ.get("OUT", "gpurun_out"), "gemm_bench.json"), "w"), indent=1)
