"""GPU: long decodes -- uniform-table refills and contexts near max_seq.

The device engines consume the reference's RandomStream uniforms
(core.py:135-179) from 4096-entry device tables with device cursors, and the
host refills a table (``consume`` + ``peek``) when a cursor nears its end
(fastpath._Tables.advance, batched._BatchRuntime.load_table).  A decode that
draws more uniforms than a table holds must still reproduce the reference
engine draw for draw.  Here the draft stream of a gamma = 32 PEARL /
SD decode crosses the table end several times, with the context running up
to within a few positions of max_seq = 4096 (the kernels' limit).
"""

from dataclasses import replace

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GAMMA = 24
PROMPT = 3600
NEW = 400
TABLE = 128


@pytest.fixture(scope="module")
def pair():
    """Tiny pair whose runtimes hold 128-entry uniform tables instead of
    4096 (fastpath.U_TABLE / batched.U_TABLE, patched before the runtimes
    exist), so a few hundred steps cross the table end many times and every
    refill (consume + peek + cursor reset) is exercised; the refill code and
    the kernels' table/cursor arguments are the production ones."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import batched, fastpath, llama
    mp = pytest.MonkeyPatch()
    mp.setattr(fastpath, "U_TABLE", TABLE)
    mp.setattr(batched, "U_TABLE", TABLE)
    yield llama.build_pair("tiny", gemm_target="tcgen05", max_seq=4096, max_tokens=64, n_slots=2,
                           align=llama.AlignSpec(branch_std=0.02))
    mp.undo()


def _prefix(seed):
    import numpy as np
    return np.random.default_rng(seed).integers(2, 32000, PROMPT).tolist()


def _strip(steps):
    keys = ("step", "kind", "drafted", "accepted_count", "correction", "finalized_delta")
    return [{k: s.to_dict()[k] for k in keys} for s in steps]


@pytest.mark.parametrize("engine", ["pearl", "sd"])
def test_long_decode_refills_tables_and_matches_reference(pair, engine):
    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    target, draft = pair
    prefix = _prefix(1)
    cfg = pk.EngineConfig(gamma=GAMMA, max_new_tokens=NEW, seed=3)
    res = (pk.decode_pearl if engine == "pearl" else pk.decode_sd)(draft, target, prefix, cfg)
    # the draft stream alone draws gamma uniforms per step: well past one table
    assert len(res.steps) * GAMMA > 3 * TABLE, len(res.steps)
    assert len(res.tokens) == NEW
    assert PROMPT + 1 + NEW + GAMMA > 4000  # the context ends near max_seq
    fn = oe.decode_pearl if engine == "pearl" else oe.decode_sd
    toks, steps = fn(draft, target, prefix, GAMMA, NEW, 3)
    assert list(res.tokens) == list(toks)
    assert _strip(res.steps) == steps


def test_long_batched_decode_equals_single(pair):
    """The batched engine's per-slot tables refill the same way: two long
    prompts in lockstep reproduce their single-prompt decodes."""
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import batched
    target, draft = pair
    prompts = [_prefix(2), _prefix(3)[:PROMPT - 40]]
    cfg = pk.EngineConfig(gamma=GAMMA, max_new_tokens=NEW, seed=9)
    got = batched.decode_pearl_batch(draft, target, prompts, cfg)
    for i, p in enumerate(prompts):
        one = pk.decode_pearl(draft, target, p, replace(cfg, seed=batched.derive_seed(cfg.seed, i)))
        assert len(one.steps) * GAMMA > 3 * TABLE
        assert got[i].tokens == one.tokens
        assert _strip(got[i].steps) == _strip(one.steps)
