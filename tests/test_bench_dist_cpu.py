"""CPU: the multi-process (N>1) plumbing of bench.py with the gloo backend.

bench.py --gpus N runs one process per GPU; each rank decodes its own prompt
shard (replicas, no data-path collective) and rank 0 reports all ranks'
tokens over the max-over-ranks time.  The aggregation and the prompt sharding
are exercised here with world_size 2 on CPU.
"""

import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", init_method="env://")
    # per-rank timed region: rank r pretends to take (r + 1) seconds for 100 tokens
    res = {"pearl": dict(device_s=float(rank + 1), event_s=float(rank + 1.5), wall_s=float(rank + 2), tokens=100 * (rank + 1))}
    agg = bench.aggregate(res, ws, device="cpu")
    prompts = bench._prompts(2, 8, 1000, seed=1000 + rank)
    q.put((rank, agg["pearl"], prompts[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_aggregation_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, (dev_max, ev_max, wall_max, tok_sum), _ in out:
        assert dev_max == 2.0 and ev_max == 2.5 and wall_max == 3.0  # max over ranks
        assert tok_sum == 300.0                                      # whole-job tokens
    assert out[0][2] != out[1][2]  # each rank decodes its own prompt shard
