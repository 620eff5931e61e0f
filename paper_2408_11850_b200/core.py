"""Value types and sampling primitives -- the reference's ``core`` API on the GPU.

Mirrors pearl_lab/core.py (names, signatures, validation, exceptions):

* ``ProbDist``     (core.py:67-120) -- host value container.  Validation and
  the one renormalisation ``probs / probs.sum()`` happen at construction,
  exactly as in the reference, so ``.probs`` is bit-identical; the CDF is
  built lazily (the device fast path never materialises ProbDists).
* ``RandomStream`` (core.py:135-179) -- PCG64 keyed by
  SeedSequence(entropy=seed, spawn_key=path), buffered so the engines can
  upload a table of future uniforms to the GPU and later consume exactly the
  draws the kernels used.
* ``sample`` (core.py:182-190) and ``residual_dist`` (core.py:193-214) run on
  the device (libpearl_b200 ``pearl_sample_rows`` / ``pearl_residual``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _device, _lib
from .errors import AllZeroResidual, InvalidDistribution, ZeroDraftProb  # noqa: F401 (re-export)

TokenId = int
TokenSeq = Tuple[TokenId, ...]

NORM_TOL = 1e-9
# The reference caps V at 65536 (core.py:24).  The B200 build serves Llama-3
# (V=128256), so the cap is raised to what the pairwise plan supports.
MAX_VOCAB = 131072
REFERENCE_MAX_VOCAB = 65536


@dataclass(frozen=True)
class Vocabulary:
    """Flat token id space with an optional reserved end-of-sequence id (core.py:39-59)."""

    size: int
    eos_id: Optional[int] = None
    token_strings: Optional[Tuple[str, ...]] = None

    def __post_init__(self) -> None:
        if not 2 <= self.size <= MAX_VOCAB:
            raise ValueError(f"vocabulary size must be in [2, {MAX_VOCAB}], got {self.size}")
        if self.eos_id is not None and not 0 <= self.eos_id < self.size:
            raise ValueError(f"eos_id {self.eos_id} outside [0, {self.size})")
        if self.token_strings is not None and len(self.token_strings) != self.size:
            raise ValueError("token_strings length must equal vocabulary size")


def byte_vocabulary() -> Vocabulary:
    """256 byte values plus a reserved EOS id (core.py:62-64)."""
    return Vocabulary(size=257, eos_id=256)


class ProbDist:
    """A validated, renormalised, immutable probability vector (core.py:67-120)."""

    __slots__ = ("probs", "_cdf_cache", "_dev")

    def __init__(self, probs) -> None:
        arr = np.asarray(probs, dtype=np.float64)
        if arr.ndim != 1:
            raise InvalidDistribution(f"expected a 1-d vector, got shape {arr.shape}")
        if not 2 <= arr.size <= MAX_VOCAB:
            raise InvalidDistribution(f"vector length {arr.size} outside [2, {MAX_VOCAB}]")
        if not np.all(np.isfinite(arr)):
            raise InvalidDistribution("probabilities must be finite")
        if np.any(arr < 0.0):
            raise InvalidDistribution(f"negative probability (min {arr.min():.3g})")
        total = float(arr.sum())
        if total == 0.0:
            raise InvalidDistribution("all-zero probability vector")
        if abs(total - 1.0) > NORM_TOL:
            raise InvalidDistribution(f"mass {total!r} is farther than {NORM_TOL} from 1")
        arr = arr / total
        arr.flags.writeable = False
        object.__setattr__(self, "probs", arr)
        object.__setattr__(self, "_cdf_cache", None)
        object.__setattr__(self, "_dev", None)

    def __setattr__(self, name: str, value: object) -> None:
        raise AttributeError("ProbDist is immutable")

    @property
    def _cdf(self) -> np.ndarray:
        """The reference's cumulative vector (core.py:98-101), built on demand."""
        if self._cdf_cache is None:
            cdf = np.cumsum(self.probs)
            cdf[-1] = 1.0
            cdf.flags.writeable = False
            object.__setattr__(self, "_cdf_cache", cdf)
        return self._cdf_cache

    def device(self, device) -> torch.Tensor:
        """The probs as a cached float64 device tensor."""
        d = self._dev
        if d is None or d.device != device:
            d = torch.from_numpy(np.array(self.probs)).to(device)
            object.__setattr__(self, "_dev", d)
        return d

    @property
    def vocab_size(self) -> int:
        return int(self.probs.size)

    def __len__(self) -> int:
        return self.vocab_size

    def __eq__(self, other: object) -> bool:
        if not hasattr(other, "probs"):
            return NotImplemented
        return bool(np.array_equal(self.probs, np.asarray(other.probs)))

    def __hash__(self):
        return id(self)

    def __repr__(self) -> str:
        return f"ProbDist(V={self.vocab_size})"


def one_hot(vocab_size: int, token: TokenId) -> ProbDist:
    v = np.zeros(vocab_size, dtype=np.float64)
    v[token] = 1.0
    return ProbDist(v)


def uniform_dist(vocab_size: int) -> ProbDist:
    return ProbDist(np.full(vocab_size, 1.0 / vocab_size))


class RandomStream:
    """Seeded splittable uniform stream (core.py:135-179), with a lookahead buffer.

    ``peek(k)`` returns the next k uniforms without consuming them and
    ``consume(k)`` advances; ``uniform()`` is peek(1) + consume(1).  The values
    are exactly those of ``Generator(PCG64(SeedSequence(seed, spawn_key=path))).random()``.
    """

    __slots__ = ("seed", "stream_id", "n_draws", "_path", "_gen", "_buf", "_pos")

    def __init__(self, seed: int, stream_id: int = 0, _path: Optional[Tuple[int, ...]] = None) -> None:
        self.seed = int(seed)
        self.stream_id = int(stream_id)
        self._path = tuple(_path) if _path is not None else (self.stream_id,)
        ss = np.random.SeedSequence(entropy=self.seed, spawn_key=self._path)
        self._gen = np.random.Generator(np.random.PCG64(ss))
        self.n_draws = 0
        self._buf = np.empty(0, dtype=np.float64)
        self._pos = 0

    def peek(self, k: int) -> np.ndarray:
        avail = self._buf.size - self._pos
        if avail < k:
            more = self._gen.random(max(k - avail, 1024))
            self._buf = np.concatenate([self._buf[self._pos:], more])
            self._pos = 0
        return self._buf[self._pos:self._pos + k]

    def consume(self, k: int) -> None:
        if k < 0 or self._pos + k > self._buf.size:
            raise ValueError("consume past the peeked window")
        self._pos += k
        self.n_draws += k

    def uniform(self) -> float:
        u = float(self.peek(1)[0])
        self.consume(1)
        return u

    def split(self, stream_id: int) -> "RandomStream":
        return RandomStream(self.seed, stream_id, _path=self._path + (int(stream_id),))

    def __repr__(self) -> str:
        return f"RandomStream(seed={self.seed}, path={self._path}, n_draws={self.n_draws})"


def split(seed: int, stream_id: int) -> RandomStream:
    return RandomStream(seed, stream_id)


def _as_probs_row(dist, device) -> torch.Tensor:
    if isinstance(dist, ProbDist):
        return dist.device(device)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(dist.probs, dtype=np.float64))).to(device)


def sample(dist, rng: RandomStream) -> TokenId:
    """Inverse-CDF sample with exactly one uniform draw, on the device (core.py:182-190)."""
    dev = _device.require_cuda()
    V = len(dist.probs)
    _lib.prepare_vocab(V)
    sc = _device.scratch()
    row = _as_probs_row(dist, dev)
    rows = _device.row_ptrs([row], dev)
    u = torch.from_numpy(np.array(rng.peek(1))).to(dev)
    out = torch.empty(1, dtype=torch.int32, device=dev)
    sc.status.zero_()
    _lib.check(_lib.load().pearl_sample_rows(
        _lib.ROWS_PROBS64, _device.ptr(rows), 1, V, _device.ptr(u), 1, None, 1.0, 0,
        _device.ptr(out), None, _device.ptr(sc.status), _device.ptr(sc.sample_work),
        _device.stream_ptr()), "sample")
    tok, st = int(out.item()), int(sc.status.item())
    _lib.check(st, "sample")
    rng.consume(1)
    return tok


def residual_dist(target, draft) -> ProbDist:
    """norm(max(target - draft, 0)) computed on the device (core.py:193-214)."""
    if len(target.probs) != len(draft.probs):
        raise InvalidDistribution(
            f"vocab mismatch: target V={len(target.probs)}, draft V={len(draft.probs)}")
    dev = _device.require_cuda()
    V = len(target.probs)
    _lib.prepare_vocab(V)
    sc = _device.scratch()
    p = _as_probs_row(target, dev)
    q = _as_probs_row(draft, dev)
    out = torch.empty(V, dtype=torch.float64, device=dev)
    sc.status.zero_()
    _lib.check(_lib.load().pearl_residual(_device.ptr(p), _device.ptr(q), V, _device.ptr(out),
                                          _device.ptr(sc.status), _device.stream_ptr()), "residual_dist")
    _lib.check(int(sc.status.item()), "residual_dist")
    return ProbDist(out.cpu().numpy())


__all__ = [
    "AllZeroResidual", "InvalidDistribution", "ZeroDraftProb", "MAX_VOCAB", "NORM_TOL", "ProbDist",
    "RandomStream", "TokenId", "TokenSeq", "Vocabulary", "byte_vocabulary", "one_hot", "residual_dist",
    "sample", "split", "uniform_dist",
]
