"""Body of __graft_entry__.smoke(): one tiny PEARL decode on cuda:0 through
the device fast path, checked against the CPU oracle.

Launches every product kernel of the decode path once or more: K2
``gemv_kernel`` (draft forward), K3 ``tc_gemm_kernel`` (target window),
K4 attention, the pick ``sample_rows_kernel``, K1 ``spec_verify_kernel`` and
the K5 ``commit_kernel``.  The oracle (oracle/engine.py, the reference engine
restated) drives the same two models through ``next_dist`` and must produce
the same tokens and StepTraces.
"""

from __future__ import annotations

import numpy as np


def _strip(steps):
    keys = ("step", "kind", "drafted", "accepted_count", "correction", "finalized_delta")
    return [{k: s.to_dict()[k] for k in keys} for s in steps]


def run_smoke() -> None:
    import torch

    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    from oracle.probdist import normalize
    from paper_2408_11850_b200 import llama

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    torch.cuda.set_device(0)

    # 1. K1 on reference-style fp64 rows vs the oracle restatement
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
    n, corr, ex = oe.verify_chain(drafted, qs, ps, oe.OracleStream(7).split(1))
    assert (res.accepted_count, res.correction, res.examined) == (n, corr, ex), (res, n, corr, ex)

    # 2. one tiny PEARL decode (T=1, gamma 4) on the fast path: tcgen05 target,
    #    CUDA-core draft; tokens and traces == the restated reference engine
    target, draft = llama.build_pair("tiny", gemm_target="tcgen05", max_seq=256, max_tokens=32)
    prefix = list(range(100, 132))
    L, gamma, seed = 24, 4, 5
    cfg = pk.EngineConfig(gamma=gamma, max_new_tokens=L, seed=seed)
    got = pk.decode_pearl(draft, target, prefix, cfg)
    assert got.stats.get("launches", 0) > 0, "decode did not take the device fast path"
    toks, steps = oe.decode_pearl(draft, target, prefix, gamma, L, seed)
    assert list(got.tokens) == list(toks), (got.tokens, toks)
    assert _strip(got.steps) == steps
    # greedy: PEARL walks the target's argmax chain (AR on the same kernels)
    gcfg = pk.EngineConfig(gamma=gamma, max_new_tokens=L, seed=seed, greedy=True)
    ar = pk.decode_autoregressive(target, prefix, gcfg).tokens
    assert pk.decode_pearl(draft, target, prefix, gcfg).tokens == ar
    torch.cuda.synchronize()
    print(f"smoke: K1 verify matches oracle {res}; tiny PEARL decode ({len(got.tokens)} tokens, "
          f"{len(got.steps)} steps, {got.stats['launches']} launches) == oracle engine; greedy PEARL == AR")
