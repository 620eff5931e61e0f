"""GPU: model-forward and decode parity at the BASELINE architectures.

Reduced-depth, FULL-WIDTH variants of every BASELINE pair (llama.pair_configs
keeps d, heads, KV heads, FFN, vocabulary and RoPE theta and cuts only the
layer count), so every kernel shape the bench runs is checked against the
oracle (oracle/llama.py):

  llama2-7b / llama-68m  head_dim 128 MHA, V 32000, theta 1e4; the 68M at full depth
  dsc-33b / dsc-1.3b     H56 / KV8 (GQA 7:1), V 32256, theta 1e5
  llama3-70b / llama3-8b H64 / KV8 and H32 / KV8 (GQA 8:1), V 128256, theta 5e5

Stated tolerances (max over a row of |logit_gpu - logit_oracle|, scaled by
the row's max |logit|; u = 2^-9 is bf16's unit roundoff):

  * LOGITS_REL_BF16 = 4u: oracle rounds to bf16 at the kernels' own points
    (and applies RMSNorm like the engine, ``norm_fold``), so only fp32
    accumulation order and transcendental ulps differ;
  * LOGITS_REL_FP32 = 8u: pure fp32 oracle -- the GPU's bf16 operands (x, q,
    k, v, attention output, SwiGLU output) each carry up to u relative error.

The residual branches use the standard init std (0.02, ``align``) so the
attention and MLP contribute O(1) to the logits instead of being hidden under
the shared bigram table.  Reference bar for the decode tests:
tests/test_engines.py:71-88 (greedy: every engine walks the target's argmax
chain) and the SequenceModel contract, models.py:58-71.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

U = 2.0 ** -9
LOGITS_REL_BF16 = 4 * U
LOGITS_REL_FP32 = 8 * U

PAIRS = [("llama2-7b/68m", (2, 2)), ("dsc-33b/1.3b", (2, 2)), ("llama3-70b/8b", (2, 2))]
N_TOK = 300


def _build(pair, depth, gemm_target="tcgen05", max_seq=640):
    from paper_2408_11850_b200 import llama
    return llama.build_pair(pair, depth=depth, gemm_target=gemm_target, max_seq=max_seq, max_tokens=128,
                            align=llama.AlignSpec(branch_std=0.02))


@pytest.fixture(scope="module", params=PAIRS, ids=[p for p, _ in PAIRS])
def pair(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.backends.cuda.matmul.allow_tf32 = False
    t, d = _build(*request.param)
    yield t, d
    del t, d
    torch.cuda.empty_cache()


def _oracle(m, bf16_points):
    from oracle.llama import OracleLlama
    return OracleLlama(m.cfg, m.w, device="cuda", bf16_points=bf16_points, max_seq=m.max_seq,
                       norm_fold=m.gemm == "tcgen05")


def _check_logits(m, toks):
    got = m.forward_logits(toks)
    for b, rel in ((True, LOGITS_REL_BF16), (False, LOGITS_REL_FP32)):
        want = _oracle(m, b).forward(toks, 0)
        scale = want.abs().amax(-1, keepdim=True)
        err = ((got - want).abs() / scale).amax(-1)
        worst = int(err.argmax())
        assert float(err.max()) <= rel, (m.cfg.name, m.gemm, "bf16 points" if b else "fp32", worst, float(err.max()))
        torch.cuda.empty_cache()


def test_logits_vs_oracle(pair):
    """Every model of every BASELINE pair, prefill windows of 128 then 128
    then 44 tokens, positions 0..299."""
    rng = np.random.default_rng(0)
    for m in pair:
        _check_logits(m, [m.bos_id] + rng.integers(0, m.cfg.vocab, N_TOK - 1).tolist())


@pytest.mark.parametrize("name", ["llama2-7b/68m", "llama3-70b/8b"])
def test_logits_vs_oracle_cudacore_target(name):
    """The CUDA-core GEMV engine (K2) as the target engine, at full width."""
    depth = dict(PAIRS)[name]
    t, d = _build(name, depth, gemm_target="cudacore")
    rng = np.random.default_rng(1)
    _check_logits(t, [t.bos_id] + rng.integers(0, t.cfg.vocab, 120).tolist())
    del t, d
    torch.cuda.empty_cache()


def _one_by_one(m, toks, start_logits_at):
    """Logits of positions start.. computed with M=1 forwards over the prefix."""
    pos = torch.zeros(1, dtype=torch.int32, device="cuda")
    t = torch.tensor(toks, dtype=torch.int32, device="cuda")
    out = torch.empty(len(toks) - start_logits_at, m.cfg.vocab, dtype=torch.float32, device="cuda")
    m.forward(t[:start_logits_at], start_logits_at, pos, 1, None)
    for j in range(start_logits_at, len(toks)):
        m.forward(t[j:j + 1], 1, pos, 1 | 2, out[j - start_logits_at:j - start_logits_at + 1])
    return out


@pytest.mark.parametrize("start,M", [(150, 5), (253, 6), (40, 16), (510, 3)])
def test_batch_invariance_bitwise(pair, start, M):
    """A window of M tokens at positions start..start+M-1 gives bitwise the
    logits of M single-token forwards."""
    rng = np.random.default_rng(start)
    for m in pair:
        toks = [m.bos_id] + rng.integers(0, m.cfg.vocab, start + M - 1).tolist()
        ref = _one_by_one(m, toks, start)
        pos = torch.zeros(1, dtype=torch.int32, device="cuda")
        t = torch.tensor(toks, dtype=torch.int32, device="cuda")
        m.forward(t[:start], start, pos, 1, None)
        win = torch.empty(M, m.cfg.vocab, dtype=torch.float32, device="cuda")
        m.forward(t[start:], M, pos, 0, win)
        assert torch.equal(win, ref), (m.cfg.name, start, M, float((win - ref).abs().max()))
        m.reset_adapter()


@pytest.mark.parametrize("start,M", [(1020, 6), (2045, 5)])
def test_batch_invariance_long_context(start, M):
    """Windows crossing the 1024-position attention super-segment boundaries
    (the cross-CTA fold of K4) stay bitwise equal to single-token forwards,
    and match the oracle; GQA 7:1 (dsc-33b width), one layer."""
    t, d = _build("dsc-33b/1.3b", (1, 1), max_seq=2100)
    rng = np.random.default_rng(start)
    for m in (t, d):
        toks = [m.bos_id] + rng.integers(0, m.cfg.vocab, start + M - 1).tolist()
        ref = _one_by_one(m, toks, start)
        pos = torch.zeros(1, dtype=torch.int32, device="cuda")
        tt = torch.tensor(toks, dtype=torch.int32, device="cuda")
        m.forward(tt[:start], start, pos, 1, None)
        win = torch.empty(M, m.cfg.vocab, dtype=torch.float32, device="cuda")
        m.forward(tt[start:], M, pos, 0, win)
        assert torch.equal(win, ref), (m.cfg.name, start, M)
        want = _oracle(m, True).forward(toks, 0)[start:]
        err = ((win - want).abs() / want.abs().amax(-1, keepdim=True)).amax()
        assert float(err) <= LOGITS_REL_BF16, (m.cfg.name, float(err))
        m.reset_adapter()
    del t, d
    torch.cuda.empty_cache()


def test_greedy_all_engines_walk_the_target_chain(pair):
    """tests/test_engines.py:71-88 at the BASELINE shapes: GPU AR == SD ==
    PEARL (gamma 4, 8, serial and concurrent) == the restated reference AR
    loop on the model's next_dist; and the chain is the fp32 oracle's argmax
    chain wherever the oracle is not within its tolerance of a tie."""
    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    target, draft = pair
    rng = np.random.default_rng(5)
    prefix = rng.integers(2, target.cfg.vocab, 64).tolist()
    L = 48
    want, _ = oe.decode_autoregressive(target, prefix, L, seed=0, greedy=True)
    for gamma in (4, 8):
        cfg = pk.EngineConfig(gamma=gamma, max_new_tokens=L, seed=3, greedy=True)
        assert pk.decode_autoregressive(target, prefix, cfg).tokens == tuple(want)
        assert pk.decode_sd(draft, target, prefix, cfg).tokens == tuple(want)
        assert pk.decode_pearl(draft, target, prefix, cfg).tokens == tuple(want)
        assert pk.decode_pearl(draft, target, prefix, cfg, concurrent=False).tokens == tuple(want)
    # teacher-forced fp32 oracle over the GPU chain
    seq = [target.bos_id] + prefix + list(want)
    lg = _oracle(target, False).forward(seq[:-1], 0)[len(prefix):]
    top = lg.argmax(-1).tolist()
    for i, (a, b) in enumerate(zip(top, want)):
        if a != b:
            gap = float(lg[i, a] - lg[i, b])
            assert gap <= LOGITS_REL_FP32 * float(lg[i].abs().max()) * 2, (i, a, b, gap)


def _strip(steps):
    keys = ("step", "kind", "drafted", "accepted_count", "correction", "finalized_delta")
    return [{k: s.to_dict()[k] for k in keys} for s in steps]


@pytest.mark.parametrize("gamma", [4, 8])
def test_sampled_step_for_step_vs_reference_engine(pair, gamma):
    """T=1: fast-path PEARL / SD tokens AND StepTraces equal the restated
    reference engines (oracle/engine.py, pinned to pearl_lab's own traces)
    driving the same models through next_dist."""
    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    target, draft = pair
    prefix = list(range(300, 340))
    L = 40
    for seed in (0, 7):
        cfg = pk.EngineConfig(gamma=gamma, max_new_tokens=L, seed=seed)
        toks, steps = oe.decode_pearl(draft, target, prefix, gamma, L, seed)
        res = pk.decode_pearl(draft, target, prefix, cfg)
        assert list(res.tokens) == list(toks) and _strip(res.steps) == steps
        toks, steps = oe.decode_sd(draft, target, prefix, gamma, L, seed)
        res = pk.decode_sd(draft, target, prefix, cfg)
        assert list(res.tokens) == list(toks) and _strip(res.steps) == steps


def test_full_depth_7b_68m_greedy_identity():
    """Full-depth Llama-2-7B / 68M (the bench pair, 13.6 GB): greedy AR ==
    SD == PEARL == the restated reference AR loop, 128 new tokens."""
    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    from paper_2408_11850_b200 import llama
    torch.cuda.empty_cache()
    target, draft = llama.build_pair("llama2-7b/68m", gemm_target="tcgen05", max_seq=512, max_tokens=128)
    rng = np.random.default_rng(11)
    prefix = rng.integers(2, 32000, 128).tolist()
    L = 128
    want, _ = oe.decode_autoregressive(target, prefix, L, seed=0, greedy=True)
    cfg = pk.EngineConfig(gamma=4, max_new_tokens=L, seed=1, greedy=True)
    assert pk.decode_autoregressive(target, prefix, cfg).tokens == tuple(want)
    assert pk.decode_sd(draft, target, prefix, cfg).tokens == tuple(want)
    assert pk.decode_pearl(draft, target, prefix, cfg).tokens == tuple(want)
    acfg = pk.EngineConfig(gamma=4, max_new_tokens=L, seed=1, greedy=True, adaptive_gamma=True, gamma_max=16)
    assert pk.decode_pearl(draft, target, prefix, acfg).tokens == tuple(want)
    del target, draft
    torch.cuda.empty_cache()
