"""CPU restatement of the reference decode loops (TEST ORACLE / CPU BASELINE ONLY).

Restates, function for function, the hot path of
``/root/reference/pkg/src/pearl_lab``:

* ``OracleStream``        -- RandomStream (core.py:135-179): PCG64 keyed by
                             SeedSequence(entropy=seed, spawn_key=path).
* ``accept_prob``         -- sampling.py:24-41
* ``verify_chain``        -- sampling.py:61-93 (+ VerifyResult sampling.py:44-58)
* ``verify_chain_greedy`` -- engines.py:220-226
* ``draft_block``         -- engines.py:265-283
* ``decode_autoregressive`` -- engines.py:289-319
* ``decode_sd``           -- engines.py:344-394 (commit rule engines.py:322-341)
* ``decode_pearl``        -- engines.py:532-591 with the pre-/post-verify
                             steps of engines.py:397-526 inlined as
                             ``_pre_step`` / ``_post_step``.

Models are duck-typed: ``model.next_dist(prefix)`` must return an object with
a float64 ``.probs`` vector that already obeys ProbDist normalisation (the
reference's ProbDist, this repo's ProbDist, or a GPU model adapter).  CDFs are
rebuilt here from ``.probs`` exactly as ProbDist does (cumsum + top guard).
Traces are plain dicts with the reference's StepTrace.to_dict keys
(engines.py:122-132), minus the abstract latencies.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from .probdist import (
    OracleZeroDraftProb,
    residual,
    sample_index,
)


class OracleStream:
    """RandomStream restated (core.py:135-179)."""

    def __init__(self, seed: int, path=(0,)):
        self.seed = int(seed)
        self.path = tuple(int(p) for p in path)
        ss = np.random.SeedSequence(entropy=self.seed, spawn_key=self.path)
        self._gen = np.random.Generator(np.random.PCG64(ss))
        self.n_draws = 0

    def uniform(self) -> float:
        self.n_draws += 1
        return float(self._gen.random())

    def split(self, stream_id: int) -> "OracleStream":
        return OracleStream(self.seed, self.path + (int(stream_id),))


def _cdf(probs: np.ndarray) -> np.ndarray:
    c = np.cumsum(np.asarray(probs, dtype=np.float64))
    c[-1] = 1.0
    return c


def sample(probs: np.ndarray, rng: OracleStream) -> int:
    """core.sample (core.py:182-190) on an already-normalised vector."""
    return sample_index(_cdf(probs), rng.uniform())


def accept_prob(p_probs: np.ndarray, q_probs: np.ndarray, token: int) -> float:
    q = float(q_probs[token])
    if q <= 0.0:
        raise OracleZeroDraftProb(f"draft probability of token {token} is {q}")
    p = float(p_probs[token])
    return 1.0 if p >= q else p / q


def verify_chain(drafted, q_rows, p_rows, rng: OracleStream):
    """Returns (accepted_count, correction or None, examined)."""
    if not (len(drafted) == len(q_rows) == len(p_rows)):
        raise ValueError("length mismatch")
    for i, tok in enumerate(drafted):
        a = accept_prob(p_rows[i], q_rows[i], tok)
        if rng.uniform() <= a:
            continue
        rprobs, rcdf = residual(np.asarray(p_rows[i]), np.asarray(q_rows[i]))
        return i, sample_index(rcdf, rng.uniform()), i + 1
    return len(drafted), None, len(drafted)


def verify_chain_greedy(drafted, p_rows):
    for i, tok in enumerate(drafted):
        best = int(np.argmax(p_rows[i]))
        if tok != best:
            return i, best, i + 1
    return len(drafted), None, len(drafted)


def _verify(drafted, q_rows, p_rows, rng, greedy):
    if greedy:
        return verify_chain_greedy(drafted, p_rows)
    return verify_chain(drafted, q_rows, p_rows, rng)


def _pick(probs, rng, greedy) -> int:
    if greedy:
        return int(np.argmax(probs))
    return sample(probs, rng)


def draft_block(draft, context, gamma, rng_draft, greedy):
    xs: List[int] = []
    qs: List[np.ndarray] = []
    buf = list(context)
    for _ in range(gamma):
        q = np.asarray(draft.next_dist(buf).probs)
        x = _pick(q, rng_draft, greedy)
        xs.append(x)
        qs.append(q)
        buf.append(x)
    return xs, qs


def _trace(index, kind, drafted, accepted, correction, delta):
    return {
        "step": index,
        "kind": kind,
        "drafted": [int(t) for t in drafted],
        "accepted_count": int(accepted),
        "correction": None if correction is None else int(correction),
        "finalized_delta": int(delta),
    }


def decode_autoregressive(target, prefix, max_new_tokens, seed, greedy=False, eos_id=None):
    rng = OracleStream(seed)
    seq = list(prefix)
    n0 = len(prefix)
    steps = []
    while len(seq) - n0 < max_new_tokens:
        tok = _pick(np.asarray(target.next_dist(seq).probs), rng, greedy)
        seq.append(tok)
        steps.append(_trace(len(steps), "ar", (), 0, None, 1))
        if eos_id is not None and tok == eos_id:
            break
    return tuple(seq[n0:]), steps


def _commit(seq, n0, block, max_new_tokens, eos_id):
    appended = 0
    for tok in block:
        seq.append(tok)
        appended += 1
        if eos_id is not None and tok == eos_id:
            return appended, True
        if len(seq) - n0 >= max_new_tokens:
            return appended, True
    return appended, False


def decode_sd(draft, target, prefix, gamma, max_new_tokens, seed, greedy=False, eos_id=None):
    root = OracleStream(seed)
    rng_d, rng_v = root.split(0), root.split(1)
    seq = list(prefix)
    n0 = len(prefix)
    steps = []
    done = False
    while not done and len(seq) - n0 < max_new_tokens:
        base = len(seq)
        xs, qs = draft_block(draft, seq, gamma, rng_d, greedy)
        window = seq + xs
        ps = [np.asarray(target.next_dist(window[: base + i]).probs) for i in range(gamma + 1)]
        n, corr, _ = _verify(xs, qs, ps[:gamma], rng_v, greedy)
        block = list(xs[:n])
        block.append(_pick(ps[gamma], rng_v, greedy) if corr is None else corr)
        appended, done = _commit(seq, n0, block, max_new_tokens, eos_id)
        steps.append(_trace(len(steps), "sd", xs, min(n, appended), corr, appended))
    return tuple(seq[n0:]), steps


def _pre_step(draft, target, committed, gamma, rng_d, rng_v, greedy, index):
    xs, qs = draft_block(draft, committed, gamma, rng_d, greedy)
    p0 = np.asarray(target.next_dist(committed).probs)
    n, corr, _ = _verify(xs[:1], qs[:1], [p0], rng_v, greedy)
    if corr is None:
        state = (tuple(committed) + (xs[0],), tuple(xs[1:]), tuple(qs[1:]), "post")
        tr = _trace(index, "pre_verify", xs, 1, None, 1)
    else:
        state = (tuple(committed) + (corr,), (), (), "pre")
        tr = _trace(index, "pre_verify", xs, 0, corr, 1)
    return state, tr


def _post_step(draft, target, committed, pending, pending_q, gamma, rng_d, rng_v, greedy, index):
    k = len(pending)
    full = list(committed) + list(pending)
    xs, qs = draft_block(draft, full, gamma, rng_d, greedy)
    ps = [np.asarray(target.next_dist(full[: len(committed) + j]).probs) for j in range(k + 1)]
    chain = list(pending) + [xs[0]]
    chain_q = list(pending_q) + [qs[0]]
    n, corr, _ = _verify(chain, chain_q, ps, rng_v, greedy)
    if corr is None:
        state = (tuple(committed) + tuple(chain), tuple(xs[1:]), tuple(qs[1:]), "post")
        tr = _trace(index, "post_verify", xs, k + 1, None, k + 1)
    else:
        state = (tuple(committed) + tuple(chain[:n]) + (corr,), (), (), "pre")
        tr = _trace(index, "post_verify", xs, n, corr, n + 1)
    return state, tr


def decode_pearl(draft, target, prefix, gamma, max_new_tokens, seed, greedy=False,
                 eos_id=None, gamma_schedule: Optional[Sequence[int]] = None):
    """decode_pearl restated; ``gamma_schedule`` (optional) gives the draft
    length per step index, for checking the adaptive-gamma extension."""
    root = OracleStream(seed)
    rng_d, rng_v = root.split(0), root.split(1)
    n0 = len(prefix)
    committed, pending, pending_q, mode = tuple(prefix), (), (), "pre"
    steps = []
    produced = 0
    while produced < max_new_tokens:
        g = gamma if gamma_schedule is None else int(gamma_schedule[len(steps)])
        if mode == "pre":
            (committed, pending, pending_q, mode), tr = _pre_step(
                draft, target, committed, g, rng_d, rng_v, greedy, len(steps))
        else:
            (committed, pending, pending_q, mode), tr = _post_step(
                draft, target, committed, pending, pending_q, g, rng_d, rng_v, greedy, len(steps))
        block = committed[n0 + produced:]
        stop = None
        if eos_id is not None:
            for off, tok in enumerate(block):
                if tok == eos_id:
                    stop = produced + off + 1
                    break
        if stop is None:
            if len(committed) - n0 >= max_new_tokens:
                stop = max_new_tokens
        else:
            stop = min(stop, max_new_tokens)
        if stop is not None:
            tr["finalized_delta"] = stop - produced
            steps.append(tr)
            return tuple(committed[n0:n0 + stop]), steps
        steps.append(tr)
        produced = len(committed) - n0
    return tuple(committed[n0:]), steps
