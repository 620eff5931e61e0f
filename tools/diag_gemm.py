import torch, sys
sys.path.insert(0, '.')
from paper_2408_11850_b200 import _lib
lib = _lib.load()
def run(N, K, M, splits=0, tag=""):
    g = torch.Generator(device="cuda").manual_seed(1)
    W = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    X = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    Y = torch.full((M, N), float('nan'), device="cuda")
    rc = lib.pearl_gemm(1, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, splits, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = X.float() @ W.float().T
    err = (Y - ref).abs()
    print(tag, N, K, M, "rc", rc, "maxerr", err.max().item(), "nan", torch.isnan(Y).sum().item(), flush=True)
for N, K in [(300, 200), (300, 256), (256, 200), (128, 200), (384, 64), (128, 128), (128, 192), (256, 64), (256, 128)]:
    for M in (1, 5, 16, 17, 64):
        run(N, K, M)
