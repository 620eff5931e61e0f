"""GPU: the plugin path of the engines reproduces the reference's traces.

Golden traces come from pearl_lab itself (make_golden.py).  Here the same
fixture models (alpha pair, hash-keyed laws, the Figure-3 scripted pair) run
through this package's engines, whose picks and verifications are CUDA
kernels; tokens and StepTraces must be identical.
"""

import numpy as np
import pytest

import recipes
from conftest import load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2408_11850_b200 as pk
    return pk


def _models(pk, run):
    if run["model"] == "alpha":
        pair = pk.make_alpha_pair(run["alpha"], vocab_size=run["V"])
        return pair.draft, pair.target
    if run["model"] == "scripted":
        v = 16
        d = {1: 1, 2: 4, 3: 5, 4: 6, 5: 7, 6: 8, 7: 9, 8: 10, 9: 11, 10: 12}
        t = {1: 13, 2: 4, 3: 5, 4: 6, 5: 7, 6: 8, 7: 14, 8: 14}
        return (pk.ScriptedModel({n: pk.one_hot(v, x) for n, x in d.items()}, vocab_size=v),
                pk.ScriptedModel({n: pk.one_hot(v, x) for n, x in t.items()}, vocab_size=v))
    V, tkw, dkw = recipes.HASH_PAIRS[run["model"]]

    class Hash(pk.SequenceModel):
        def __init__(self, lat, kw):
            self.vocab_size, self.latency, self.kw, self.cache = V, pk.LatencyProfile(lat), kw, {}

        def next_dist(self, prefix):
            key = tuple(prefix)
            if key not in self.cache:
                self.cache[key] = pk.ProbDist(recipes.hash_probs(V, prefix=prefix, **self.kw))
            return self.cache[key]
    return Hash(1.0, dkw), Hash(3.0, tkw)


def _check(res, want):
    assert list(res.tokens) == want["tokens"]
    assert [s.to_dict() for s in res.steps] == want["steps"]


def test_plugin_engines_match_reference_traces(pk):
    runs = load_golden("engine_traces.json")
    for i, run in enumerate(runs):
        if run["model"] == "alpha" and i % 3:   # thin the alpha grid to keep the test quick
            continue
        draft, target = _models(pk, run)
        cfg = pk.EngineConfig(gamma=run["gamma"], max_new_tokens=run["L"], seed=run["seed"],
                              greedy=run["greedy"], eos_id=run["eos"])
        _check(pk.decode_pearl(draft, target, run["prefix"], cfg, concurrent=False), run["pearl"])
        if "sd" in run:
            _check(pk.decode_sd(draft, target, run["prefix"], cfg), run["sd"])
            _check(pk.decode_autoregressive(target, run["prefix"], cfg), run["ar"])


def test_concurrent_matches_serial_plugin(pk):
    V, tkw, dkw = recipes.HASH_PAIRS["hash64"]
    runs = load_golden("engine_traces.json")
    run = next(r for r in runs if r["model"] == "hash64" and not r["greedy"])
    draft, target = _models(pk, run)
    cfg = pk.EngineConfig(gamma=run["gamma"], max_new_tokens=run["L"], seed=run["seed"])
    a = pk.decode_pearl(draft, target, run["prefix"], cfg, concurrent=False)
    b = pk.decode_pearl(draft, target, run["prefix"], cfg, concurrent=True)
    assert a == b


def test_lossless_point_mass(pk):
    pair = pk.make_alpha_pair(0.6, vocab_size=32)
    cfg = pk.EngineConfig(gamma=3, max_new_tokens=40, seed=5)
    assert pk.decode_pearl(pair.draft, pair.target, [], cfg, concurrent=False).tokens == (0,) * 40
    assert pk.decode_sd(pair.draft, pair.target, [], cfg).tokens == (0,) * 40
