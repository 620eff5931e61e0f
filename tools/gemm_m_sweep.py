"""Back-to-back timing of the tcgen05 GEMM over token counts M (epilogue / MMA scaling)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import _lib
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
for N, K in ((22016, 4096), (4096, 11008), (12288, 4096)):
    W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    row = []
    for M in (1, 4, 16, 32, 48, 64, 96, 128):
        X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Y = torch.empty(M, N, device="cuda")
        f = lambda: lib.pearl_gemm(1, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, 0, st)
        for _ in range(3): f()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(20): f()
        e.record(); e.synchronize()
        t = s.elapsed_time(e) / 20 * 1e3
        row.append(f"M={M}:{t:.1f}us({N*K*2/t/1e3:.0f}GB/s)")
    print(f"N={N} K={K}: " + " ".join(row), flush=True)
