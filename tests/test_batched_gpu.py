"""GPU: batched lockstep decoding (batched.py).

The reference has no batching; its CLI decodes a prompt list as independent
decodes with per-prompt derived seeds (cli.py:94-96).  The bar: decoding B
prompts together returns, for every prompt, exactly the tokens AND StepTraces
of the single-prompt engine with that prompt's seed -- PEARL, SD and AR,
greedy and sampled (T=1), ragged prompt lengths, EOS mid-batch.  This holds
because every kernel is batch invariant (a token's logits are bitwise the
same whichever tokens share the launch, tests/test_llama_gpu.py).
"""

from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

PROMPTS = [[5, 17, 300, 9, 44, 1203, 77, 8], [900, 31, 2, 2, 2, 64], [12, 13], list(range(100, 131))]


@pytest.fixture(scope="module", params=["tcgen05", "cudacore"])
def pair(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import llama
    return llama.build_pair("tiny", gemm_target=request.param, max_seq=256, max_tokens=32, n_slots=len(PROMPTS))


def _strip(res):
    return (tuple(res.tokens),
            tuple((t.kind, tuple(t.drafted), t.accepted_count, t.correction, t.finalized_delta) for t in res.steps))


def _single(engine, draft, target, cfg, i):
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200.batched import derive_seed
    c = replace(cfg, seed=derive_seed(cfg.seed, i))
    if engine == "pearl":
        return pk.decode_pearl(draft, target, PROMPTS[i], c)
    if engine == "sd":
        return pk.decode_sd(draft, target, PROMPTS[i], c)
    return pk.decode_autoregressive(target, PROMPTS[i], c)


def _batch(engine, draft, target, cfg):
    from paper_2408_11850_b200 import batched
    if engine == "pearl":
        return batched.decode_pearl_batch(draft, target, PROMPTS, cfg)
    if engine == "sd":
        return batched.decode_sd_batch(draft, target, PROMPTS, cfg)
    return batched.decode_autoregressive_batch(target, PROMPTS, cfg)


@pytest.mark.parametrize("engine", ["pearl", "sd", "ar"])
@pytest.mark.parametrize("greedy", [True, False])
def test_batch_equals_independent_decodes(pair, engine, greedy):
    import paper_2408_11850_b200 as pk
    target, draft = pair
    cfg = pk.EngineConfig(gamma=4, max_new_tokens=40, seed=3, greedy=greedy)
    got = _batch(engine, draft, target, cfg)
    assert len(got) == len(PROMPTS)
    for i, r in enumerate(got):
        want = _single(engine, draft, target, cfg, i)
        assert _strip(r) == _strip(want), (engine, greedy, i)


def test_batch_eos_mid_batch(pair):
    import paper_2408_11850_b200 as pk
    target, draft = pair
    base = pk.EngineConfig(gamma=3, max_new_tokens=30, seed=8, greedy=False)
    for engine in ("pearl", "sd", "ar"):
        # EOS = a token prompt 1 produces early, so one sequence stops while the others run on
        eos = _single(engine, draft, target, base, 1).tokens[2]
        cfg = replace(base, eos_id=int(eos))
        got = _batch(engine, draft, target, cfg)
        for i, r in enumerate(got):
            assert _strip(r) == _strip(_single(engine, draft, target, cfg, i)), (engine, i)
        assert any(len(r.tokens) < cfg.max_new_tokens for r in got)


def test_forward_slots_matches_single_sequence(pair):
    """Slot-mode logits of mixed sequences == single-sequence logits, bitwise."""
    target, _ = pair
    rng = np.random.default_rng(0)
    seqs = [[target.bos_id] + rng.integers(0, target.cfg.vocab, n).tolist() for n in (9, 4, 13)]
    singles = [target.forward_logits(s) for s in seqs]
    toks, slots, pos = [], [], []
    for i, s in enumerate(seqs):
        toks += s
        slots += [i] * len(s)
        pos += list(range(len(s)))
    dev = target.device
    t = torch.tensor(toks, dtype=torch.int32, device=dev)
    sl = torch.tensor(slots, dtype=torch.int32, device=dev)
    p = torch.tensor(pos, dtype=torch.int32, device=dev)
    out = torch.empty(len(toks), target.cfg.vocab, dtype=torch.float32, device=dev)
    target.forward_slots(t, len(toks), sl, p, out)
    off = 0
    for s, want in zip(seqs, singles):
        assert torch.equal(out[off:off + len(s)], want)
        off += len(s)
