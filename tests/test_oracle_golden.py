"""CPU: pin the oracle restatement against the reference's own outputs.

The golden files were produced by the reference package itself
(tests/golden/make_golden.py); these tests need no GPU.
"""

import numpy as np
import pytest

import recipes
from conftest import load_golden
from oracle import engine as oe
from oracle import probdist as op


class _Dist:
    def __init__(self, probs):
        self.probs, _ = op.normalize(probs)


# -- pairwise summation tree (what the device emulates) ----------------------


@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 257, 1000, 4095, 4096, 8193, 32000, 32256])
def test_pairwise_tree_equals_numpy_sum(n):
    rng = np.random.default_rng(n)
    a = rng.random(n) ** 5 * 10.0 ** rng.integers(-3, 3)
    assert op.pairwise_sum_tree(a) == float(a.sum())


def test_cumsum_is_sequential():
    a = np.random.default_rng(0).random(5000)
    c = np.cumsum(a)
    run = 0.0
    for i, x in enumerate(a):
        run = run + x
        assert run == c[i]


# -- device exp / logits law ---------------------------------------------------


def test_dev_expf_accuracy_and_edges():
    x = np.linspace(-79.9, 0.0, 200001, dtype=np.float32)
    e = op.dev_expf(x)
    ref = np.exp(x.astype(np.float64))
    assert np.max(np.abs(e - ref) / ref) < 2.5e-7
    assert op.dev_expf(np.float32([0.0]))[0] == 1.0
    assert op.dev_expf(np.float32([-np.inf, -81.0, -1e30]))[:].tolist() == [0.0, 0.0, 0.0]
    assert np.all(np.diff(op.dev_expf(x)) >= 0)  # monotone


def test_logits_law_is_valid_probdist():
    for V in (2, 257, 32000):
        l = recipes.make_logits(V, 1, V)[0]
        p1 = op.logits_to_p1(l, 1.0)
        probs, cdf = op.normalize(p1)
        assert cdf[-1] == 1.0 and abs(p1.sum() - 1.0) < 1e-12


# -- verify_chain / greedy ------------------------------------------------------


def test_verify_cases_against_reference():
    g = load_golden("verify_cases.json")
    for case in g["cases"]:
        ps, qs = recipes.make_rows(case["V"], case["n"], case["seed"], case["kind"])
        P = [_Dist(p) for p in ps]
        Q = [_Dist(q) for q in qs]
        assert recipes.sha(*[d.probs for d in P]) == case["sha_p"]
        assert recipes.sha(*[d.probs for d in Q]) == case["sha_q"]
        root = oe.OracleStream(case["seed"] + case["rng_seed"])
        rd, rv = root.split(0), root.split(1)
        drafted = [oe.sample(q.probs, rd) for q in Q]
        assert drafted == case["drafted"]
        assert [oe.OracleStream(case["seed"] + case["rng_seed"]).split(1).uniform() for _ in range(1)] \
            == case["u_head"][:1]
        acc = [oe.accept_prob(P[i].probs, Q[i].probs, drafted[i]) for i in range(case["n"])]
        assert acc == case["accept_probs"]
        n, corr, ex = oe.verify_chain(drafted, [q.probs for q in Q], [p.probs for p in P], rv)
        assert case["error"] is None
        assert (n, -1 if corr is None else corr, ex, rv.n_draws) == (
            case["accepted"], case["correction"], case["examined"], case["n_draws"])
        gn, gc, _ = oe.verify_chain_greedy(drafted, [p.probs for p in P])
        assert (gn, -1 if gc is None else gc) == (case["g_accepted"], case["g_correction"])


class _Stub:
    def __init__(self, us):
        self.us, self.n_draws = list(us), 0

    def uniform(self):
        u = self.us[self.n_draws]
        self.n_draws += 1
        return u


def test_verify_edge_cases_against_reference():
    g = load_golden("verify_cases.json")
    errs = {"AllZeroResidual": op.OracleAllZeroResidual, "ZeroDraftProb": op.OracleZeroDraftProb}
    for case in g["edges"]:
        P = [op.normalize(r)[0] for r in case["p"]]
        Q = [op.normalize(r)[0] for r in case["q"]]
        rng = _Stub(case["uniforms"])
        if case["error"]:
            with pytest.raises(errs[case["error"]]):
                oe.verify_chain(case["drafted"], Q, P, rng)
            assert rng.n_draws == case["n_draws"], case["name"]
        else:
            n, corr, ex = oe.verify_chain(case["drafted"], Q, P, rng)
            assert (n, -1 if corr is None else corr, ex, rng.n_draws) == (
                case["accepted"], case["correction"], case["examined"], case["n_draws"]), case["name"]


def test_sample_cases_against_reference():
    for case in load_golden("sample_cases.json"):
        ps, _ = recipes.make_rows(case["V"], 1, case["seed"], case["kind"])
        probs, cdf = op.normalize(ps[0])
        assert recipes.sha(probs) == case["sha"]
        for u, want in zip(case["us"], case["idx"]):
            assert op.sample_index(cdf, u) == want
            assert op.sample_index_seq(probs, u) == want


def test_residual_cases_against_reference():
    for case in load_golden("residual_cases.json"):
        ps, qs = recipes.make_rows(case["V"], 1, case["seed"], case["kind"])
        p, _ = op.normalize(ps[0])
        q, _ = op.normalize(qs[0])
        r, cdf = op.residual(p, q)
        assert recipes.sha(r) == case["sha_r"]
        assert [op.sample_index(cdf, u) for u in case["us"]] == case["idx"]


def test_logits_cases_against_reference():
    for case in load_golden("logits_cases.json"):
        lp = recipes.make_logits(case["V"], case["n"], case["seed"], kind=case["kind"])
        lq = recipes.make_logits(case["V"], case["n"], case["seed"] + 1, kind=case["kind"])
        P = [op.logits_to_probs(r, case["inv_t"])[0] for r in lp]
        Q = [op.logits_to_probs(r, case["inv_t"])[0] for r in lq]
        assert recipes.sha(*P) == case["sha_p"]
        root = oe.OracleStream(case["seed"] * 3 + case["rng_seed"])
        rd, rv = root.split(0), root.split(1)
        drafted = [oe.sample(q, rd) for q in Q]
        assert drafted == case["drafted"]
        n, corr, ex = oe.verify_chain(drafted, Q, P, rv)
        assert (n, -1 if corr is None else corr, ex, rv.n_draws) == (
            case["accepted"], case["correction"], case["examined"], case["n_draws"])
        assert [int(np.argmax(p)) for p in P] == case["argmax"]


# -- engines ------------------------------------------------------------------


class _AlphaModel:
    def __init__(self, probs):
        self.d = _Dist(probs)

    def next_dist(self, prefix):
        return self.d


class _HashModel:
    def __init__(self, V, **kw):
        self.V, self.kw = V, kw

    def next_dist(self, prefix):
        return _Dist(recipes.hash_probs(self.V, prefix=prefix, **self.kw))


class _Scripted:
    def __init__(self, table, V):
        self.table, self.V = table, V

    def next_dist(self, prefix):
        v = np.zeros(self.V)
        v[self.table[len(prefix)]] = 1.0
        return _Dist(v)


def _models(run):
    if run["model"] == "alpha":
        a, V = run["alpha"], run["V"]
        q = np.full(V, (1.0 - a) / (V - 1))
        q[0] = a
        t = np.zeros(V)
        t[0] = 1.0
        return _AlphaModel(q), _AlphaModel(t)
    if run["model"] == "scripted":
        draft = {1: 1, 2: 4, 3: 5, 4: 6, 5: 7, 6: 8, 7: 9, 8: 10, 9: 11, 10: 12}
        target = {1: 13, 2: 4, 3: 5, 4: 6, 5: 7, 6: 8, 7: 14, 8: 14}
        return _Scripted(draft, 16), _Scripted(target, 16)
    V, tkw, dkw = recipes.HASH_PAIRS[run["model"]]
    return _HashModel(V, **dkw), _HashModel(V, **tkw)


def _strip(steps):
    keys = ("step", "kind", "drafted", "accepted_count", "correction", "finalized_delta")
    return [{k: s[k] for k in keys} for s in steps]


def test_engine_traces_against_reference():
    for run in load_golden("engine_traces.json"):
        draft, target = _models(run)
        kw = dict(greedy=run["greedy"], eos_id=run["eos"])
        toks, steps = oe.decode_pearl(draft, target, run["prefix"], run["gamma"], run["L"], run["seed"], **kw)
        assert list(toks) == run["pearl"]["tokens"]
        assert steps == _strip(run["pearl"]["steps"])
        if "sd" in run:
            toks, steps = oe.decode_sd(draft, target, run["prefix"], run["gamma"], run["L"], run["seed"], **kw)
            assert list(toks) == run["sd"]["tokens"] and steps == _strip(run["sd"]["steps"])
            toks, steps = oe.decode_autoregressive(target, run["prefix"], run["L"], run["seed"], **kw)
            assert list(toks) == run["ar"]["tokens"] and steps == _strip(run["ar"]["steps"])
