"""Deterministic input recipes shared by the golden generator and the tests.

``make_golden.py`` (run in the build container, where the reference package
``pearl_lab`` is importable from /root/reference) feeds these inputs to the
reference and records its outputs; the tests regenerate the same inputs from
the same recipes (numpy only) and compare the oracle / the CUDA kernels with
the recorded outputs.  Each case also stores a SHA-256 of its inputs so a
drift in regeneration is caught instead of silently comparing other data.
"""

from __future__ import annotations

import hashlib
from typing import List, Sequence, Tuple

import numpy as np

# -- probability rows ---------------------------------------------------------


def _normed(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x / x.sum()


def make_rows(V: int, n: int, seed: int, kind: str) -> Tuple[List[np.ndarray], List[np.ndarray]]:
    """n (p, q) row pairs of length V.  kinds:

    random   -- independent peaky random laws (acceptance ~ 0.3-0.6)
    close    -- q a small perturbation of p (acceptance ~ 0.9+)
    sparse   -- both laws supported on a few hundred ids with zeros elsewhere
    disjoint -- p and q with disjoint supports (certain rejection)
    equal    -- p == q (certain acceptance)
    """
    rng = np.random.default_rng(seed)
    ps, qs = [], []
    for _ in range(n):
        if kind == "random":
            p = _normed(rng.random(V) ** 8)
            q = _normed(rng.random(V) ** 8)
        elif kind == "close":
            p = _normed(rng.random(V) ** 8)
            q = _normed(p * (1.0 + 0.2 * rng.random(V)))
        elif kind == "sparse":
            p = np.zeros(V)
            q = np.zeros(V)
            m = max(2, min(V, 300))
            p[rng.choice(V, m, replace=False)] = rng.random(m)
            q[rng.choice(V, m, replace=False)] = rng.random(m)
            common = rng.choice(V, 1)
            p[common] += 1.0
            q[common] += 1.0
            p, q = _normed(p), _normed(q)
        elif kind == "disjoint":
            half = V // 2
            p = np.zeros(V)
            q = np.zeros(V)
            p[:half] = rng.random(half) + 0.1
            q[half:] = rng.random(V - half) + 0.1
            p, q = _normed(p), _normed(q)
        elif kind == "equal":
            p = _normed(rng.random(V) ** 4)
            q = p.copy()
        else:
            raise ValueError(kind)
        ps.append(p)
        qs.append(q)
    return ps, qs


def make_logits(V: int, n: int, seed: int, scale: float = 4.0, kind: str = "gauss") -> np.ndarray:
    """fp32 logits rows [n, V] for the logits-mode kernels."""
    rng = np.random.default_rng(seed)
    if kind == "gauss":
        return (rng.standard_normal((n, V)) * scale).astype(np.float32)
    if kind == "ties":  # many exact ties at the maximum
        x = np.round(rng.standard_normal((n, V)) * 2.0).astype(np.float32)
        return x
    if kind == "masked":  # -inf entries (banned tokens) and a large spread
        x = (rng.standard_normal((n, V)) * scale).astype(np.float32)
        x[:, rng.random(V) < 0.3] = -np.inf
        x[:, 0] = 0.0
        return x
    raise ValueError(kind)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


# -- a prefix-keyed pseudo-random model pair (engine traces) -------------------


def hash_probs(V: int, seed: int, prefix: Sequence[int], ctx: int = 3, sharp: float = 3.0,
               noise: float = 0.0, noise_seed: int = 0) -> np.ndarray:
    """A pure prefix -> law map: softmax of Gaussian logits keyed by the last
    ``ctx`` tokens.  ``noise`` adds an independent perturbation (draft model)."""
    tail = [int(t) for t in prefix[-ctx:]]
    key = [seed, len(prefix) % 7] + tail
    rng = np.random.default_rng(np.random.SeedSequence(entropy=key))
    logits = rng.standard_normal(V) * sharp
    if noise > 0.0:
        nrng = np.random.default_rng(np.random.SeedSequence(entropy=[noise_seed] + key))
        logits = logits + nrng.standard_normal(V) * noise
    e = np.exp(logits - logits.max())
    return e / e.sum()


HASH_PAIRS = {
    # name: (V, target kwargs, draft kwargs)
    "hash64": (64, dict(seed=11, sharp=2.5), dict(seed=11, sharp=2.5, noise=0.8, noise_seed=5)),
    "hash300": (300, dict(seed=23, sharp=3.0), dict(seed=23, sharp=3.0, noise=1.2, noise_seed=9)),
}
