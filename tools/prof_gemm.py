"""Run one GEMM shape a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import _lib
N, K, M, kind = (int(x) for x in sys.argv[1:5])
lib = _lib.load()
W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Y = torch.empty(M, N, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    lib.pearl_gemm(kind, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, 0, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
