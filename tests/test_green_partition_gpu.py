"""GPU: PEARL with the draft on its own green-context SM partition (the
bench's default for the 68M draft).  The target's stream-K grids shrink to
its partition for every engine, so greedy AR == SD == PEARL still hold token
for token, and sampled PEARL / SD / AR still reproduce the restated
reference engines step for step (as tests/test_llama_gpu.py checks on
shared SMs)."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def green_pair():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2408_11850_b200 import llama
    target, draft = llama.build_pair("tiny", gemm_target="tcgen05", max_seq=512, max_tokens=32, draft_sms=16)
    if getattr(target, "green_partition", None) is None:
        pytest.skip("green contexts unavailable on this driver")
    return target, draft


def _strip(steps):
    keys = ("step", "kind", "drafted", "accepted_count", "correction", "finalized_delta")
    return [{k: s.to_dict()[k] for k in keys} for s in steps]


def test_partition_sizes(green_pair):
    target, draft = green_pair
    ds, ts, nd, nt = target.green_partition
    assert nd >= 16 and nt >= 1 and nd + nt <= torch.cuda.get_device_properties(0).multi_processor_count


def test_greedy_identity_on_partition(green_pair):
    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    target, draft = green_pair
    prefix = list(range(5, 21))
    want, _ = oe.decode_autoregressive(target, prefix, 40, seed=0, greedy=True)
    for gamma in (1, 4):
        cfg = pk.EngineConfig(gamma=gamma, max_new_tokens=40, seed=3, greedy=True)
        assert pk.decode_autoregressive(target, prefix, cfg).tokens == tuple(want)
        assert pk.decode_sd(draft, target, prefix, cfg).tokens == tuple(want)
        assert pk.decode_pearl(draft, target, prefix, cfg).tokens == tuple(want)


def test_sampled_parity_on_partition(green_pair):
    import paper_2408_11850_b200 as pk
    from oracle import engine as oe
    target, draft = green_pair
    prefix = list(range(100, 116))
    for gamma in (2, 4):
        cfg = pk.EngineConfig(gamma=gamma, max_new_tokens=48, seed=7)
        toks, steps = oe.decode_pearl(draft, target, prefix, gamma, 48, 7)
        res = pk.decode_pearl(draft, target, prefix, cfg)
        assert list(res.tokens) == list(toks) and _strip(res.steps) == steps
    cfg = pk.EngineConfig(gamma=3, max_new_tokens=48, seed=9, adaptive_gamma=True, gamma_max=16)
    res = pk.decode_pearl(draft, target, prefix, cfg)
    toks, steps = oe.decode_pearl(draft, target, prefix, 3, 48, 9, gamma_schedule=res.stats["gammas"])
    assert list(res.tokens) == list(toks) and _strip(res.steps) == steps
