"""The model plugin boundary (pearl_lab/models.py) and the small fixture models.

* ``LatencyProfile`` (models.py:42-55) and the ``SequenceModel`` ABC
  (models.py:58-71) are the drop-in point: anything with
  ``next_dist(prefix) -> ProbDist``, ``vocab_size`` and ``latency`` plugs into
  the engines, exactly as in the reference.
* GPU models (``paper_2408_11850_b200.llama.LlamaModel``) are SequenceModels
  too (their ``next_dist`` is an adapter over the device forward), and they
  additionally implement the device fast-path protocol the engines detect
  (``is_device_model``).
* ``ConstDistModel`` / ``AlphaPair`` / ``ScriptedModel`` (models.py:232-296)
  are the reference's exact-answer fixtures, kept for parity tests.
"""

from __future__ import annotations

from abc import ABC, abstractmethod
from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .core import ProbDist, TokenId, one_hot
from .errors import InvalidAlpha


@dataclass(frozen=True)
class LatencyProfile:
    """Cost of one forward pass (abstract units, or measured seconds for GPU models)."""

    forward_time: float = 1.0

    def __post_init__(self) -> None:
        if not self.forward_time > 0.0:
            raise ValueError(f"forward_time must be positive, got {self.forward_time}")


class SequenceModel(ABC):
    """Anything that maps a token prefix to a next-token distribution."""

    vocab_size: int
    latency: LatencyProfile

    @abstractmethod
    def next_dist(self, prefix: Sequence[TokenId]) -> ProbDist:
        """The next-token distribution after ``prefix`` (pure in ``prefix``)."""


def is_device_model(m) -> bool:
    """True for models that implement the device fast path (llama.LlamaModel)."""
    return bool(getattr(m, "_pearl_device_model", False))


class ConstDistModel(SequenceModel):
    """Same distribution for every prefix (models.py:232-241)."""

    def __init__(self, dist: ProbDist, latency: LatencyProfile | None = None) -> None:
        self._dist = dist
        self.vocab_size = dist.vocab_size
        self.latency = latency if latency is not None else LatencyProfile()

    def next_dist(self, prefix: Sequence[TokenId]) -> ProbDist:
        return self._dist


@dataclass(frozen=True)
class AlphaPair:
    """Draft/target pair with constant per-token acceptance alpha (models.py:244-259)."""

    alpha: float
    draft: SequenceModel
    target: SequenceModel


def make_alpha_pair(alpha: float, vocab_size: int = 64, draft_time: float = 1.0,
                    target_time: float = 1.0) -> AlphaPair:
    """Point-mass target on token 0, draft alpha on 0 (models.py:262-280)."""
    if not 0.0 <= alpha <= 1.0:
        raise InvalidAlpha(f"alpha must be in [0, 1], got {alpha}")
    if vocab_size < 2:
        raise ValueError(f"vocab_size must be >= 2, got {vocab_size}")
    probs = np.full(vocab_size, (1.0 - alpha) / (vocab_size - 1))
    probs[0] = alpha
    draft = ConstDistModel(ProbDist(probs), LatencyProfile(draft_time))
    target = ConstDistModel(one_hot(vocab_size, 0), LatencyProfile(target_time))
    return AlphaPair(alpha=alpha, draft=draft, target=target)


@dataclass
class ScriptedModel(SequenceModel):
    """Prefix-length -> distribution table for forced traces (models.py:283-296)."""

    table: Mapping[int, ProbDist]
    vocab_size: int
    latency: LatencyProfile = field(default_factory=LatencyProfile)

    def next_dist(self, prefix: Sequence[TokenId]) -> ProbDist:
        n = len(prefix)
        try:
            return self.table[n]
        except KeyError:
            raise KeyError(f"no scripted distribution for prefix length {n}") from None


def estimate_alpha(draft: SequenceModel, target: SequenceModel, prefixes) -> float:
    """Mean sum(min(p, q)) over prefixes (models.py:299-316)."""
    if len(prefixes) == 0:
        raise ValueError("need at least one prefix")
    total = 0.0
    for prefix in prefixes:
        p = np.asarray(target.next_dist(prefix).probs)
        q = np.asarray(draft.next_dist(prefix).probs)
        total += float(np.minimum(p, q).sum())
    return total / len(prefixes)


def compute_c(draft_latency: LatencyProfile, target_latency: LatencyProfile) -> float:
    """Target / draft forward cost ratio (models.py:319-321)."""
    return target_latency.forward_time / draft_latency.forward_time
