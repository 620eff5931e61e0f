"""GPU: the two contraction engines (K2 CUDA-core GEMV, K3 tcgen05+TMA) vs a
plain PyTorch fp32 reference of the same op, and their batch invariance."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SHAPES = [(128, 64), (300, 200), (2752, 512), (512, 1376), (4096, 4096), (12288, 4096), (32000, 768),
          (4096, 11008), (1000, 72)]


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _lib
    return _lib


def _gemm(lib, kind, W, X, splits=0, N=None):
    M, K = X.shape
    N = W.shape[0] if N is None else N
    Y = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    lib.check(lib.load().pearl_gemm(kind, W.data_ptr(), X.data_ptr(), Y.data_ptr(), M, N, K, splits,
                                    torch.cuda.current_stream().cuda_stream), "pearl_gemm")
    torch.cuda.synchronize()
    return Y


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("N,K", SHAPES)
def test_matches_fp32_reference(lib, kind, N, K):
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K)
    W = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    for M in (1, 3, 16, 17, 40, 64, 100, 128):
        X = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
        Y = _gemm(lib, kind, W, X)
        ref = X.float() @ W.float().T
        tol = 2e-5 * K ** 0.5 + 1e-4 * ref.abs().max().item()
        assert torch.isfinite(Y).all()
        assert (Y - ref).abs().max().item() <= tol, (kind, N, K, M, (Y - ref).abs().max().item())


@pytest.mark.parametrize("kind", [0, 1])
def test_batch_invariance(lib, kind):
    g = torch.Generator(device="cuda").manual_seed(5)
    shapes = [(4096, 4096), (300, 1376), (32000, 768)]
    if kind == 0:
        # K2's single-token kernel (gemv1_kernel): one chunk batch (768 / 3072: the
        # 68M draft's o / down), a 12 + 1 chunk split (3328), ragged N and K, the
        # 4-row-per-warp wide path (9999 rows) -- all bitwise the multi-token rows
        shapes += [(768, 3072), (1001, 3328), (9999, 520), (2304, 768)]
    for N, K in shapes:
        W = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
        X = torch.randn(128, K, generator=g, device="cuda").to(torch.bfloat16)
        full = _gemm(lib, kind, W, X)
        for M in (1, 2, 5, 16, 33, 64, 100):
            part = _gemm(lib, kind, W, X[:M].contiguous())
            assert torch.equal(part, full[:M]), (kind, N, K, M)
        # a token's row does not depend on the other rows' values either
        X2 = X.clone()
        X2[1:] = torch.randn_like(X2[1:].float()).to(torch.bfloat16)
        assert torch.equal(_gemm(lib, kind, W, X2)[0], full[0])


def test_split_k_is_deterministic_and_close(lib):
    g = torch.Generator(device="cuda").manual_seed(9)
    W = (torch.randn(4096, 11008, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    X = torch.randn(8, 11008, generator=g, device="cuda").to(torch.bfloat16)
    a = _gemm(lib, 1, W, X)
    assert torch.equal(a, _gemm(lib, 1, W, X))
    b = _gemm(lib, 1, W, X, splits=1)
    assert (a - b).abs().max().item() < 1e-2


@pytest.mark.parametrize("N,K", [(4096, 4096), (22016, 4096), (4096, 11008)])
def test_tile_major_weights_bitwise(lib, N, K):
    """PEARL_GEMM_W_TILED: the same weights stored tile-major ([N/128][K/64]
    [128][64], every TMA box one contiguous 16 KB) give bitwise the row-major
    result for decode and prefill windows."""
    g = torch.Generator(device="cuda").manual_seed(N + K)
    W = (torch.randn(N, K, generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    Wt = W.view(N // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous()
    for M in (1, 16, 20, 64, 128):
        X = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
        assert torch.equal(_gemm(lib, 1, W, X), _gemm(lib, 1 | 0x100, Wt, X, N=N)), (N, K, M)
