"""GPU: K5 in-place KV rollback through the C ABI (``pearl_kv_rollback``).

The reference rolls back by rebuilding DecodeState without the rejected
drafts (engines.py:500-515); the device keeps the KV cache in place and only
resets its length -- positions past the new length are overwritten by the
next window.  Inside the engines the commit kernel does this; external
callers (include/pearl_b200.h K5) use ``pearl_kv_rollback``.  The bar: after
forwarding rejected tokens and rolling back, the next window's logits are
bitwise those of a forward that never saw the rejected tokens.
"""

import ctypes

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("gemm", ["tcgen05", "cudacore"])
def test_rollback_discards_rejected_window(gemm):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _device, _lib, llama
    target, _ = llama.build_pair("tiny", gemm_target=gemm, max_seq=256, max_tokens=32)
    lib = _lib.load()
    prefix = torch.arange(40, 80, dtype=torch.int32, device="cuda")
    junk = torch.tensor([7, 7, 9, 11, 13], dtype=torch.int32, device="cuda")
    real = torch.tensor([101, 202, 303], dtype=torch.int32, device="cuda")
    V = target.cfg.vocab

    # clean: prefix, then the real window
    pos = torch.zeros(1, dtype=torch.int32, device="cuda")
    target.forward(prefix, len(prefix), pos, 1, None)
    want = torch.empty(3, V, device="cuda")
    target.forward(real, 3, pos, 0, want)

    # rejected window forwarded (and advanced), then rolled back through K5
    pos = torch.zeros(1, dtype=torch.int32, device="cuda")
    target.forward(prefix, len(prefix), pos, 1, None)
    target.forward(junk, len(junk), pos, 1, torch.empty(len(junk), V, device="cuda"))
    torch.cuda.synchronize()
    assert int(pos.item()) == len(prefix) + len(junk)
    new_len = torch.tensor([len(prefix)], dtype=torch.int32, device="cuda")
    _lib.check(lib.pearl_kv_rollback(_device.ptr(pos), _device.ptr(new_len), 1,
                                     ctypes.c_void_p(_device.stream_ptr())), "pearl_kv_rollback")
    got = torch.empty(3, V, device="cuda")
    target.forward(real, 3, pos, 0, got)
    torch.cuda.synchronize()
    assert int(pos.item()) == len(prefix)
    assert torch.equal(got, want)


def test_rollback_many_lengths():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _device, _lib
    lib = _lib.load()
    n = 1000
    lens = torch.arange(n, dtype=torch.int32, device="cuda") + 50
    new = torch.randint(0, 50, (n,), dtype=torch.int32, device="cuda")
    _lib.check(lib.pearl_kv_rollback(_device.ptr(lens), _device.ptr(new), n, ctypes.c_void_p(_device.stream_ptr())),
               "pearl_kv_rollback")
    torch.cuda.synchronize()
    assert torch.equal(lens, new)
    with pytest.raises(Exception):
        _lib.check(lib.pearl_kv_rollback(None, _device.ptr(new), n, None), "pearl_kv_rollback")
