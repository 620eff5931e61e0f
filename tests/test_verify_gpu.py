"""GPU parity of K1 (pearl_spec_verify) and the pick / law kernels.

Bit-exact against the reference's golden outputs (tests/golden) on the same
ProbDist rows and the same PCG64 uniforms, and against the oracle for the
logits-mode device law.  Everything calls through the C ABI.
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


def _probs_rows(rows):
    from oracle.probdist import normalize
    return [torch.from_numpy(np.array(normalize(r)[0])).cuda() for r in rows]


def _verify(pk, p_rows, q_rows, drafted, uniforms, flags=0, mode=0, inv_t=1.0, V=None):
    from paper_2408_11850_b200 import _device, _lib
    dev = torch.device("cuda")
    V = V or int(p_rows[0].numel())
    _lib.prepare_vocab(V)
    sc = _device.scratch()
    pr = _device.row_ptrs(p_rows, dev)
    qr = _device.row_ptrs(q_rows, dev) if q_rows else None
    toks = torch.tensor(drafted, dtype=torch.int32, device=dev)
    u = torch.tensor(np.asarray(uniforms, dtype=np.float64), device=dev) if len(uniforms) else None
    cursor = torch.zeros(1, dtype=torch.int32, device=dev)
    acc = torch.zeros(len(drafted), dtype=torch.float64, device=dev)
    code = _lib.load().pearl_spec_verify(
        mode, _device.ptr(pr), _device.ptr(qr), _device.ptr(toks), len(drafted), V, _device.ptr(u),
        0 if u is None else u.numel(), _device.ptr(cursor), inv_t, flags | _lib.F_ADVANCE,
        _device.ptr(sc.result), _device.ptr(acc), _device.ptr(sc.verify_work), _device.stream_ptr())
    _lib.check(code)
    r = sc.result.cpu().numpy().tolist()
    return dict(status=r[0], accepted=r[1], correction=r[2], examined=r[3], draws=r[4], bonus=r[5],
                fallback=r[6], cursor=int(cursor.item()), accept=acc.cpu().numpy())


def test_verify_cases_bit_exact(pk):
    g = load_golden("verify_cases.json")
    for case in g["cases"]:
        ps, qs = recipes.make_rows(case["V"], case["n"], case["seed"], case["kind"])
        P, Q = _probs_rows(ps), _probs_rows(qs)
        rv = pk.RandomStream(case["seed"] + case["rng_seed"]).split(1)
        us = rv.peek(case["n"] + 1)
        assert list(us[:3]) == case["u_head"][: len(us[:3])]
        r = _verify(pk, P, Q, case["drafted"], us)
        got = (r["status"], r["accepted"], r["correction"], r["examined"], r["draws"], r["cursor"])
        want = (0, case["accepted"], case["correction"], case["examined"], case["n_draws"], case["n_draws"])
        assert got == want, (case["V"], case["kind"], case["n"], case["rng_seed"])
        assert r["accept"].tolist() == case["accept_probs"]
        rg = _verify(pk, P, None, case["drafted"], [], flags=1)
        assert (rg["accepted"], rg["correction"], rg["draws"]) == (case["g_accepted"], case["g_correction"], 0)


def test_verify_edge_cases(pk):
    codes = {"AllZeroResidual": 2, "ZeroDraftProb": 3}
    for case in load_golden("verify_cases.json")["edges"]:
        P, Q = _probs_rows(case["p"]), _probs_rows(case["q"])
        r = _verify(pk, P, Q, case["drafted"], case["uniforms"])
        if case["error"]:
            assert r["status"] == codes[case["error"]], case["name"]
            assert r["draws"] == case["n_draws"], case["name"]
        else:
            assert (r["status"], r["accepted"], r["correction"], r["examined"], r["draws"]) == (
                0, case["accepted"], case["correction"], case["examined"], case["n_draws"]), case["name"]


def test_logits_mode_matches_reference_on_device_law(pk):
    from oracle.probdist import logits_to_p1
    from paper_2408_11850_b200 import _device, _lib
    for case in load_golden("logits_cases.json"):
        V, n = case["V"], case["n"]
        lp = recipes.make_logits(V, n, case["seed"], kind=case["kind"])
        lq = recipes.make_logits(V, n, case["seed"] + 1, kind=case["kind"])
        tp = torch.from_numpy(lp).cuda()
        tq = torch.from_numpy(lq).cuda()
        # the device law itself is bit-identical to the oracle twin
        _lib.prepare_vocab(V)
        out = torch.empty((n, V), dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(_lib.load().pearl_logits_to_probs(_device.ptr(tp), n, V, case["inv_t"],
                                                     _device.ptr(out), _device.ptr(st), _device.stream_ptr()))
        assert int(st.item()) == 0
        want = np.stack([logits_to_p1(r, case["inv_t"]) for r in lp])
        assert np.array_equal(out.cpu().numpy(), want), (V, case["kind"])
        rv = pk.RandomStream(case["seed"] * 3 + case["rng_seed"]).split(1)
        r = _verify(pk, [tp[i] for i in range(n)], [tq[i] for i in range(n)], case["drafted"],
                    rv.peek(n + 1), mode=1, inv_t=case["inv_t"], V=V)
        assert (r["status"], r["accepted"], r["correction"], r["examined"], r["draws"]) == (
            0, case["accepted"], case["correction"], case["examined"], case["n_draws"])
        rg = _verify(pk, [tp[i] for i in range(n)], None, case["drafted"], [], flags=1, mode=1,
                     inv_t=case["inv_t"], V=V)
        assert (rg["accepted"], rg["correction"]) == (case["g_accepted"], case["g_correction"])


def test_sample_cases_bit_exact(pk):
    from paper_2408_11850_b200 import _device, _lib
    for case in load_golden("sample_cases.json"):
        ps, _ = recipes.make_rows(case["V"], 1, case["seed"], case["kind"])
        row = _probs_rows(ps)[0]
        V = case["V"]
        _lib.prepare_vocab(V)
        k = len(case["us"])
        rows = _device.row_ptrs([row] * k, torch.device("cuda"))
        u = torch.tensor(case["us"], dtype=torch.float64, device="cuda")
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        work = torch.zeros(4096, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().pearl_sample_rows(0, _device.ptr(rows), k, V, _device.ptr(u), k, None, 1.0, 0,
                                                 _device.ptr(out), None, _device.ptr(st), _device.ptr(work),
                                                 _device.stream_ptr()))
        assert int(st.item()) == 0
        assert out.cpu().tolist() == case["idx"], (V, case["kind"])


def test_residual_and_api(pk):
    from oracle.probdist import normalize
    for case in load_golden("residual_cases.json"):
        ps, qs = recipes.make_rows(case["V"], 1, case["seed"], case["kind"])
        P, Q = pk.ProbDist(ps[0]), pk.ProbDist(qs[0])
        r = pk.residual_dist(P, Q)
        assert recipes.sha(r.probs) == case["sha_r"]
        for u, want in zip(case["us"][:4], case["idx"][:4]):
            class _R:
                def peek(self, k):
                    return np.array([u])

                def consume(self, k):
                    pass
            assert pk.sample(r, _R()) == want
    # API KATs (tests/test_sampling.py:11-77 of the reference)
    p = pk.ProbDist([0.6, 0.4])
    q = pk.ProbDist([0.4, 0.6])
    assert pk.accept_prob(p, q, 0) == 1.0
    assert pk.accept_prob(p, q, 1) == 0.4 / 0.6
    with pytest.raises(pk.ZeroDraftProb):
        pk.accept_prob(pk.ProbDist([0.5, 0.5, 0.0]), pk.ProbDist([0.5, 0.0, 0.5]), 1)
    d = pk.ProbDist([0.3, 0.3, 0.4])
    assert pk.verify_chain([0, 1, 2], [d] * 3, [d] * 3, pk.RandomStream(1)) == pk.VerifyResult(3, None, 3)
    res = pk.verify_chain([1], [pk.one_hot(4, 1)], [pk.one_hot(4, 3)], pk.RandomStream(0))
    assert (res.accepted_count, res.correction, res.examined) == (0, 3, 1)
    d2 = pk.ProbDist([0.5, 0.5])
    rng = pk.RandomStream(3)
    pk.verify_chain([0, 1], [d2, d2], [d2, d2], rng)
    assert rng.n_draws == 2
    rng = pk.RandomStream(3)
    pk.verify_chain([0, 0], [d2, pk.one_hot(2, 0)], [d2, pk.one_hot(2, 1)], rng)
    assert rng.n_draws == 3
    with pytest.raises(ValueError):
        pk.verify_chain([0, 1], [d2], [d2, d2], pk.RandomStream(0))
    assert pk.verify_chain([], [], [], pk.RandomStream(0)) == pk.VerifyResult(0, None, 0)
    with pytest.raises(pk.AllZeroResidual):
        pk.residual_dist(pk.ProbDist([0.25, 0.75]), pk.ProbDist([0.25, 0.75]))
    np.testing.assert_allclose(pk.residual_dist(pk.ProbDist([0.4, 0.4, 0.2]), pk.ProbDist([0.1, 0.2, 0.7])).probs,
                               [0.6, 0.4, 0.0], atol=1e-12)
    assert all(pk.sample(pk.one_hot(6, 2), pk.RandomStream(0)) == 2 for _ in range(5))
    _ = normalize


def test_empirical_law_one_slot(pk):
    """Single-slot output law == p (reference tests/test_sampling.py:80-115), 20k draws."""
    from paper_2408_11850_b200 import _device, _lib
    P, Q = [0.5, 0.3, 0.2], [0.2, 0.5, 0.3]
    rng = np.random.default_rng(42)
    N = 20000
    counts = np.zeros(3)
    p_row, q_row = _probs_rows([P, Q])
    for _ in range(N // 2000):
        us = rng.random((2000, 3))
        for k in range(2000):
            y = int(np.searchsorted(np.cumsum(Q), us[k, 0], side="right"))
            r = _verify(pk, [p_row], [q_row], [y], us[k, 1:])
            counts[y if r["accepted"] == 1 else r["correction"]] += 1
    np.testing.assert_allclose(counts / N, P, atol=0.015)


@pytest.mark.parametrize("V", [32256, 128256])
def test_large_vocab_against_oracle(pk, V):
    """V beyond the reference's MAX_VOCAB (Llama-3: 128256, 16-CTA clusters):
    K1 and the pick kernel against the oracle restatement of core.py/sampling.py
    on the device law of the same logits and the same PCG64 uniforms."""
    from oracle import engine as oe
    from oracle.probdist import logits_to_probs, sample_index
    n = 4
    for seed in (1, 2, 3):
        lp = recipes.make_logits(V, n, seed, scale=3.0)
        lq = (lp + recipes.make_logits(V, n, seed + 100, scale=0.7)).astype(np.float32)  # correlated draft
        P = [logits_to_probs(r)[0] for r in lp]
        Qd = [logits_to_probs(r) for r in lq]
        rd = oe.OracleStream(seed).split(0)
        drafted = [sample_index(cdf, rd.uniform()) for _, cdf in Qd]
        rv = oe.OracleStream(seed).split(1)
        want = oe.verify_chain(drafted, [q for q, _ in Qd], P, rv)
        us = pk.RandomStream(seed).split(1).peek(n + 1)
        tp, tq = torch.from_numpy(lp).cuda(), torch.from_numpy(lq).cuda()
        r = _verify(pk, [tp[i] for i in range(n)], [tq[i] for i in range(n)], drafted, us, mode=1, V=V)
        got = (r["accepted"], None if r["correction"] < 0 else r["correction"], r["examined"])
        assert r["status"] == 0 and got == want and r["draws"] == rv.n_draws, (V, seed, got, want)
        # probs64 mode on the oracle's normalised rows gives the same verdict
        r2 = _verify(pk, [torch.from_numpy(np.array(p)).cuda() for p in P],
                     [torch.from_numpy(np.array(q)).cuda() for q, _ in Qd], drafted, us)
        assert (r2["accepted"], r2["correction"], r2["draws"]) == (r["accepted"], r["correction"], r["draws"])
    # inverse-CDF pick at adversarial uniforms (exact cdf values and neighbours)
    from paper_2408_11850_b200 import _device, _lib
    probs, cdf = logits_to_probs(recipes.make_logits(V, 1, 77, scale=2.0)[0])
    rng = np.random.default_rng(5)
    us = [0.0, float(np.nextafter(1.0, 0.0))]
    for i in rng.choice(V - 1, 8, replace=False):
        c = float(cdf[i])
        us += [c, float(np.nextafter(c, 0.0)), float(np.nextafter(c, 2.0))]
    us = [u for u in us if 0.0 <= u < 1.0]
    row = torch.from_numpy(np.array(probs)).cuda()
    rows = _device.row_ptrs([row] * len(us), torch.device("cuda"))
    u = torch.tensor(us, dtype=torch.float64, device="cuda")
    out = torch.empty(len(us), dtype=torch.int32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    work = torch.zeros(65536, dtype=torch.uint8, device="cuda")
    _lib.prepare_vocab(V)
    _lib.check(_lib.load().pearl_sample_rows(0, _device.ptr(rows), len(us), V, _device.ptr(u), len(us), None, 1.0, 0,
                                             _device.ptr(out), None, _device.ptr(st), _device.ptr(work),
                                             _device.stream_ptr()))
    assert int(st.item()) == 0
    assert out.cpu().tolist() == [sample_index(cdf, x) for x in us]


def _verify_multi(chains, V, flags, mode=0, inv_t=1.0, tail=False):
    """pearl_spec_verify_multi over `chains` = [(P rows, Q rows or None, drafted, uniforms)] in ONE
    launch; with tail=True each chain's last id is read through the descriptor's tail pointer."""
    from paper_2408_11850_b200 import _device, _lib
    dev = torch.device("cuda")
    _lib.prepare_vocab(V)
    bonus = bool(flags & _lib.F_BONUS)
    keep, words, base = [], [], 0
    wb = int(_lib.load().pearl_verify_work_bytes(max(len(c[2]) for c in chains) + 1))
    outs = torch.zeros(len(chains), 8, dtype=torch.int32, device=dev)
    curs = torch.zeros(len(chains), dtype=torch.int32, device=dev)
    work = torch.zeros(len(chains), wb, dtype=torch.uint8, device=dev)
    for i, (P, Q, drafted, us) in enumerate(chains):
        pr = _device.row_ptrs(P, dev)
        qr = _device.row_ptrs(Q, dev) if Q else pr
        ids = list(drafted) + [-7]  # a poisoned slot after the chain
        if tail:
            ids[len(drafted) - 1] = -5  # must be read through `tail` instead
        toks = torch.tensor(ids, dtype=torch.int32, device=dev)
        tl = torch.tensor([drafted[-1]], dtype=torch.int32, device=dev)
        u = torch.tensor(np.asarray(us, dtype=np.float64), device=dev) if len(us) else None
        keep += [pr, qr, toks, tl, u]
        n = len(drafted)
        words.append([pr.data_ptr(), qr.data_ptr(), toks.data_ptr(), tl.data_ptr() if tail else 0,
                      0 if u is None else u.data_ptr(), curs[i:].data_ptr(), outs[i].data_ptr(),
                      work[i].data_ptr(), n | (base << 32), 1])
        base += n + (1 if bonus else 0)
    d = torch.tensor(np.array(words, np.int64).reshape(-1), device=dev)
    n_u = max(len(c[3]) for c in chains)
    _lib.check(_lib.load().pearl_spec_verify_multi(mode, _device.ptr(d), len(chains), base, V, n_u, inv_t,
                                                   flags | _lib.F_ADVANCE, _device.stream_ptr()))
    torch.cuda.synchronize()
    o = outs.cpu().numpy()
    c = curs.cpu().numpy()
    return [dict(status=int(r[0]), accepted=int(r[1]), correction=int(r[2]), examined=int(r[3]), draws=int(r[4]),
                 bonus=int(r[5]), cursor=int(ci)) for r, ci in zip(o, c)]


def test_verify_multi_equals_per_chain(pk):
    """One batched K1 launch == pearl_spec_verify per chain (golden verdicts), mixed
    chain lengths, sampled / greedy / SD bonus, ids via the tail pointer."""
    from paper_2408_11850_b200 import _lib
    g = load_golden("verify_cases.json")
    by_v = {}
    for case in g["cases"]:
        by_v.setdefault(case["V"], []).append(case)
    for V, cases in by_v.items():
        cases = cases[:12]
        chains, singles = [], []
        for case in cases:
            ps, qs = recipes.make_rows(case["V"], case["n"], case["seed"], case["kind"])
            P, Q = _probs_rows(ps), _probs_rows(qs)
            us = pk.RandomStream(case["seed"] + case["rng_seed"]).split(1).peek(case["n"] + 2)
            chains.append((P, Q, case["drafted"], us))
            singles.append((0, case["accepted"], case["correction"], case["examined"], case["n_draws"]))
        for tail in (False, True):
            got = _verify_multi(chains, V, 0, tail=tail)
            assert [(r["status"], r["accepted"], r["correction"], r["examined"], r["draws"]) for r in got] == singles
            assert [r["cursor"] for r in got] == [s[4] for s in singles]
        got = _verify_multi([(P, None, d, []) for P, _, d, _ in chains], V, _lib.F_GREEDY)
        assert [(r["accepted"], r["correction"]) for r in got] == [(c["g_accepted"], c["g_correction"]) for c in cases]
        # SD bonus: p has one more row; compare with the single-chain kernel on the same rows
        bon = [(P + [P[0]], Q, d, us) for P, Q, d, us in chains]
        got = _verify_multi(bon, V, _lib.F_BONUS)
        for (P, Q, d, us), r in zip(bon, got):
            want = _verify(pk, P, Q, d, us, flags=_lib.F_BONUS)
            assert (r["status"], r["accepted"], r["correction"], r["bonus"], r["draws"]) == (
                want["status"], want["accepted"], want["correction"], want["bonus"], want["draws"])
