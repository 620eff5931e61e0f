"""GPU: the split pair (draft and target on different devices, one process
each, K6 mailboxes over CUDA IPC) reproduces the co-resident fast path.

This box has one GPU, so both ranks run on cuda:0 as two processes (CUDA IPC
maps the mailboxes within one device exactly as across NVLink peers; the
handshake goes over gloo).  On an 8-GPU box the same code runs with each rank
on its own device.  The bar: tokens and StepTraces (kind, drafted,
accepted_count, correction, finalized_delta) identical to co-resident
decode_pearl on the same seeds -- greedy and sampled (T=1), fixed gamma --
and, with adaptive gamma, both ranks return the same result and greedy
tokens equal the target's AR decode.
"""

import os
import socket
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROMPTS = [[5, 17, 300, 9, 44, 1203, 77, 8], [900, 31, 2, 2, 2, 64]]
NEW = 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _strip(res):
    return (tuple(res.tokens),
            tuple((t.kind, tuple(t.drafted), t.accepted_count, t.correction, t.finalized_delta) for t in res.steps))


def _cases():
    import paper_2408_11850_b200 as pk
    out = []
    for greedy in (True, False):
        for i, pr in enumerate(PROMPTS):
            out.append((pr, pk.EngineConfig(gamma=4, max_new_tokens=NEW, seed=11 + i, greedy=greedy,
                                            gamma_max=8)))
    out.append((PROMPTS[0], pk.EngineConfig(gamma=3, max_new_tokens=NEW, seed=5, greedy=True,
                                            adaptive_gamma=True, gamma_max=8)))
    return out


def _worker(rank, port, q, mode="peer_store"):
    try:
        sys.path.insert(0, REPO)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE="2")
        if mode == "copy_engine":
            os.environ["PEARL_K6_COPY"] = "1"
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method="env://")
        import paper_2408_11850_b200 as pk
        from paper_2408_11850_b200 import llama, split_pair as split
        role, peer = split.pair_roles(rank, 2)
        target, draft = llama.build_pair("tiny", gemm_target="tcgen05", max_seq=256, max_tokens=32)
        local = target if role == split.ROLE_TARGET else draft
        remote = split.connect_pair(local, role, peer, gamma_max=8, timeout_s=60.0)
        assert remote.link.mode == mode, remote.link.mode
        outs = []
        for pr, cfg in _cases():
            if role == split.ROLE_TARGET:
                r = pk.decode_pearl(remote, target, pr, cfg)
            else:
                r = pk.decode_pearl(draft, remote, pr, cfg)
            outs.append(_strip(r))
        remote.link.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, outs, None))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


@pytest.fixture(scope="module", params=["peer_store", "copy_engine"])
def split_results(request):
    """Both K6 transports: direct peer stores (NVLink / same device) and the
    copy-engine fallback for GPUs that cannot map each other (forced here
    with PEARL_K6_COPY=1)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, request.param)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, outs, err = q.get(timeout=600)
        assert err is None, f"rank {rank}:\n{err}"
        got[rank] = outs
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


def test_both_ranks_agree(split_results):
    assert split_results[0] == split_results[1]


def test_split_matches_coresident(split_results):
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import llama
    target, draft = llama.build_pair("tiny", gemm_target="tcgen05", max_seq=256, max_tokens=32)
    for (pr, cfg), got in zip(_cases(), split_results[0]):
        if cfg.adaptive_gamma:
            ar = pk.decode_autoregressive(target, pr, cfg)
            assert got[0] == tuple(ar.tokens)
            continue
        want = _strip(pk.decode_pearl(draft, target, pr, cfg))
        assert got == want, (cfg, got[0], want[0])


def test_exchange_wait_times_out_instead_of_hanging():
    """A K6 wait whose peer never pushes reports PEARL_ERR_TIMEOUT (DeviceError
    at the Python layer) after its timeout instead of spinning forever."""
    import ctypes
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _lib
    lib = _lib.load()
    box = ctypes.c_void_p()
    _lib.check(lib.pearl_mailbox_alloc(int(lib.pearl_mailbox_bytes(0, 8)), ctypes.byref(box)), "alloc")
    try:
        ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        dst = torch.zeros(8, dtype=torch.int32, device="cuda")
        _lib.check(lib.pearl_xfer_wait(box, ctr.data_ptr() + 8, dst.data_ptr(), 8, status.data_ptr(),
                                       int(0.2e9), torch.cuda.current_stream().cuda_stream), "wait")
        torch.cuda.synchronize()
        assert int(status.item()) == _lib.PEARL_ERR_TIMEOUT
        assert int(ctr[1].item()) == 1  # the receive sequence still advanced (lockstep)
    finally:
        lib.pearl_mailbox_free(box)


def test_exchange_push_then_wait_same_process():
    """One push into a (locally mapped) mailbox, then the wait returns the ids."""
    import ctypes
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _lib, split_pair
    lib = _lib.load()
    V = 64
    box = ctypes.c_void_p()
    _lib.check(lib.pearl_mailbox_alloc(int(lib.pearl_mailbox_bytes(3, V)), ctypes.byref(box)), "alloc")
    try:
        ctr = torch.zeros(3, dtype=torch.int64, device="cuda")  # send, recv, arrive
        ids = torch.arange(5, dtype=torch.int32, device="cuda") + 7
        rows = torch.randn(3, V, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        a = split_pair._XferArgs(box.value, ids.data_ptr(), 5, rows.data_ptr(), 3, V, ctr.data_ptr(), ctr.data_ptr() + 16)
        _lib.check(lib.pearl_xfer_send(ctypes.byref(a), st), "send")
        dst = torch.zeros(5, dtype=torch.int32, device="cuda")
        status = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(lib.pearl_xfer_wait(box, ctr.data_ptr() + 8, dst.data_ptr(), 5, status.data_ptr(), int(5e9), st),
                   "wait")
        torch.cuda.synchronize()
        assert int(status.item()) == 0 and torch.equal(dst, ids)
        assert ctr[0].item() == 1 and ctr[1].item() == 1 and ctr[2].item() == 0
        got = torch.empty(3 * V, dtype=torch.float32)
        cu = ctypes.CDLL("libcuda.so.1")  # driver API: read the raw mailbox rows back
        cu.cuMemcpyDtoH_v2.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t]
        assert cu.cuMemcpyDtoH_v2(got.data_ptr(), box.value + _lib.MAILBOX_ROWS_OFFSET, 3 * V * 4) == 0
        assert torch.equal(got.view(3, V), rows.cpu())
    finally:
        lib.pearl_mailbox_free(box)


def test_exchange_copy_engine_push_then_wait():
    """The copy-engine push (pearl_xfer_send_copy) delivers ids, rows and the
    sequence flag in order, like the peer-store kernel."""
    import ctypes
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _lib, split_pair
    lib = _lib.load()
    V = 48
    box = ctypes.c_void_p()
    _lib.check(lib.pearl_mailbox_alloc(int(lib.pearl_mailbox_bytes(2, V)), ctypes.byref(box)), "alloc")
    try:
        ctr = torch.zeros(4, dtype=torch.int64, device="cuda")  # send, recv, arrive, staging
        st = torch.cuda.current_stream().cuda_stream
        for it in range(3):
            ids = torch.arange(4, dtype=torch.int32, device="cuda") + 100 * it
            rows = torch.randn(2, V, device="cuda")
            a = split_pair._XferArgs(box.value, ids.data_ptr(), 4, rows.data_ptr(), 2, V, ctr.data_ptr(),
                                     ctr.data_ptr() + 16)
            _lib.check(lib.pearl_xfer_send_copy(ctypes.byref(a), ctr.data_ptr() + 24, st), "send_copy")
            dst = torch.zeros(4, dtype=torch.int32, device="cuda")
            status = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.check(lib.pearl_xfer_wait(box, ctr.data_ptr() + 8, dst.data_ptr(), 4, status.data_ptr(), int(5e9),
                                           st), "wait")
            torch.cuda.synchronize()
            assert int(status.item()) == 0 and torch.equal(dst, ids)
            assert ctr[0].item() == it + 1 and ctr[1].item() == it + 1 and ctr[3].item() == it + 1
    finally:
        lib.pearl_mailbox_free(box)


def test_peer_storable_same_device():
    import ctypes
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import _lib
    lib = _lib.load()
    bus = ctypes.create_string_buffer(64)
    _lib.check(lib.pearl_pci_bus_id(bus, 64), "pci")
    assert lib.pearl_peer_storable(bus.value) == 1
    assert lib.pearl_peer_storable(b"0000:ff:1f.0") == 0  # not a visible device
