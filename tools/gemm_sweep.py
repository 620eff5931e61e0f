"""Back-to-back timing of the tcgen05 GEMM (stream-K) for a shape over grid sizes G and M."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import _lib
lib = _lib.load()
N, K = int(sys.argv[1]), int(sys.argv[2])
W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for M in (1, 4, 16):
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(M, N, device="cuda")
    res = []
    for S in (74, 96, 128, 148, 0):
        f = lambda: lib.pearl_gemm(1, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, S, st)
        for _ in range(3): f()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(20): f()
        e.record(); e.synchronize()
        t = s.elapsed_time(e) / 20 * 1e3
        res.append(f"G={S if S else 'auto'}:{t:.1f}us/{N*K*2/t/1e3:.0f}GB/s")
    print(f"N={N} K={K} M={M}: " + "  ".join(res), flush=True)
