"""CPU: host-side logic of the split pair (split_pair.py) with world_size-2 gloo.

The K6 kernels need a GPU (tests/test_split_gpu.py); here the handshake
(entry exchange + role / vocabulary / gamma_max checks), the rank -> role
mapping and the shared adaptive-gamma planner are exercised across two real
processes.
"""

import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeLink:
    def __init__(self, role, peer_info):
        self.role, self.peer_info = role, peer_info


def _worker(rank, ws, port, bad, q):
    try:
        sys.path.insert(0, REPO)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
        dist.init_process_group("gloo", init_method="env://")
        from paper_2408_11850_b200 import split_pair as split
        role, peer = split.pair_roles(rank, ws)
        if role == split.ROLE_DRAFT:
            info = {"t_d": 1e-4 * (1 + rank), "latency": 1e-4}
        else:
            info = {"t_t": {1: 3e-3, 8: 3.2e-3, 16: 3.5e-3, 32: 4.5e-3}, "latency": 3e-3}
        entry = {"role": role, "rank": rank, "handle": bytes([rank]) * 64, "vocab": 32000,
                 "gamma_max": 32 + (rank if bad else 0), "info": info}
        try:
            p = split.exchange_entries(entry, peer)
        except ValueError as e:
            q.put((rank, "error", str(e)))
            dist.destroy_process_group()
            return
        planner = split._PlannerFromLink(_FakeLink(role, p["info"]), info, 32, 4)
        gammas = []
        for i in range(40):  # identical observation history on both ranks
            gammas.append(planner.next_gamma())
            planner.observe(3 if i % 5 else 0, 1 if i % 5 == 0 else 0)
        q.put((rank, "ok", (role, peer, p["rank"], p["handle"], gammas)))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "crash", traceback.format_exc()))


def _run(ws, bad=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, bad, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = dict((r, (k, v)) for r, k, v in (q.get(timeout=120) for _ in range(ws)))
    for p in procs:
        p.join(timeout=60)
    return out


def test_handshake_and_shared_planner_four_ranks():
    out = _run(4)
    for r, (kind, v) in out.items():
        assert kind == "ok", v
        role, peer, got_rank, handle, _ = v
        assert peer == (r + 1 if r % 2 == 0 else r - 1)
        assert role == ("target" if r % 2 == 0 else "draft")
        assert got_rank == peer and handle == bytes([peer]) * 64
    # each pair's two planners make the same gamma choices
    for a, b in ((0, 1), (2, 3)):
        assert out[a][1][4] == out[b][1][4]
    # pair (2,3) has a slower draft (t_d scales with the draft rank) -> its own schedule
    assert out[0][1][4] != out[2][1][4] or len(set(out[0][1][4])) == 1


def test_handshake_rejects_mismatched_gamma_max():
    out = _run(2, bad=True)
    for r, (kind, v) in out.items():
        assert kind == "error" and "gamma_max" in v


def test_pair_roles():
    from paper_2408_11850_b200 import split_pair as split
    assert [split.pair_roles(r, 8) for r in range(4)] == [("target", 1), ("draft", 0), ("target", 3), ("draft", 2)]
    with pytest.raises(ValueError):
        split.pair_roles(0, 3)
