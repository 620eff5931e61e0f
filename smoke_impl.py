"""Body of __graft_entry__.smoke(): one tiny decode on cuda:0 checked against the oracle."""

from __future__ import annotations

import numpy as np


def run_smoke() -> None:
    import torch

    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    from oracle.probdist import normalize

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    torch.cuda.set_device(0)
    # K1 on reference-style rows vs the oracle restatement
    rng = np.random.default_rng(0)
    V = 32000
    def law():
        x = rng.random(V) ** 8
        return normalize(x / x.sum())[0]
    ps = [law() for _ in range(4)]
    qs = [law() for _ in range(4)]
    drafted = [int(np.argmax(q)) for q in qs]
    res = pk.verify_chain(drafted, [pk.ProbDist(q) for q in qs], [pk.ProbDist(p) for p in ps],
                          pk.RandomStream(7).split(1))
    ors = oe.OracleStream(7).split(1)
    n, corr, ex = oe.verify_chain(drafted, qs, ps, ors)
    assert (res.accepted_count, res.correction, res.examined) == (n, corr, ex), (res, n, corr, ex)
    torch.cuda.synchronize()
    print("smoke: K1 verify matches oracle", res)
