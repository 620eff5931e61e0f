"""The lossless accept-or-resample rule, on the device (pearl_lab/sampling.py).

``accept_prob`` (sampling.py:24-41), ``VerifyResult`` (sampling.py:44-58) and
``verify_chain`` (sampling.py:61-93) keep the reference's names, argument
meaning, results, RNG consumption and exceptions; the arithmetic is the fused
K1 kernel (``pearl_spec_verify``), bit-exact with the reference on the same
ProbDist rows and uniforms.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device, _lib
from .core import ProbDist, RandomStream, TokenId, _as_probs_row


@dataclass(frozen=True)
class VerifyResult:
    accepted_count: int
    correction: Optional[TokenId]
    examined: int


def _launch_verify(drafted, draft_dists, target_dists, uniforms: np.ndarray, flags: int,
                   want_accept: bool = False):
    dev = _device.require_cuda()
    n = len(drafted)
    V = len(target_dists[0].probs)
    for d in list(draft_dists) + list(target_dists):
        if len(d.probs) != V:
            raise ValueError("all distributions of a chain must share one vocabulary")
    _lib.prepare_vocab(V)
    sc = _device.scratch()
    p_rows = _device.row_ptrs([_as_probs_row(d, dev) for d in target_dists], dev)
    q_rows = _device.row_ptrs([_as_probs_row(d, dev) for d in draft_dists], dev) if draft_dists else None
    toks = torch.tensor([int(t) for t in drafted], dtype=torch.int32, device=dev)
    u = torch.from_numpy(np.ascontiguousarray(uniforms, dtype=np.float64)).to(dev) if len(uniforms) else None
    acc = torch.zeros(n, dtype=torch.float64, device=dev) if want_accept else None
    flags_eff = flags
    bonus_rows = len(target_dists) - n
    if bonus_rows == 1:
        flags_eff |= _lib.F_BONUS
    code = _lib.load().pearl_spec_verify(
        _lib.ROWS_PROBS64, _device.ptr(p_rows), _device.ptr(q_rows), _device.ptr(toks), n, V,
        _device.ptr(u), 0 if u is None else int(u.numel()), None, 1.0, flags_eff,
        _device.ptr(sc.result), _device.ptr(acc), _device.ptr(sc.verify_work), _device.stream_ptr())
    _lib.check(code, "pearl_spec_verify")
    res = sc.result.cpu().numpy()
    return res, (acc.cpu().numpy() if acc is not None else None)


def accept_prob(target_dist: ProbDist, draft_dist: ProbDist, token: TokenId) -> float:
    """min(1, p[token]/q[token]); ZeroDraftProb if q[token] == 0 (sampling.py:24-41)."""
    res, acc = _launch_verify([token], [draft_dist], [target_dist], np.zeros(0), _lib.F_PROBE,
                              want_accept=True)
    _lib.check(int(res[0]), "accept_prob")
    return float(acc[0])


def verify_chain(
    drafted: Sequence[TokenId],
    draft_dists: Sequence[ProbDist],
    target_dists: Sequence[ProbDist],
    rng: RandomStream,
) -> VerifyResult:
    """Accept a prefix of ``drafted`` and resample at the first rejection.

    Consumes exactly ``examined`` uniforms plus one for the correction, like
    the reference (sampling.py:61-93).
    """
    if not (len(drafted) == len(draft_dists) == len(target_dists)):
        raise ValueError(
            f"length mismatch: {len(drafted)} drafts, {len(draft_dists)} draft dists, "
            f"{len(target_dists)} target dists")
    n = len(drafted)
    if n == 0:
        return VerifyResult(accepted_count=0, correction=None, examined=0)
    res, _ = _launch_verify(drafted, draft_dists, target_dists, rng.peek(n + 1), 0)
    status, accepted, correction, examined, draws = (int(x) for x in res[:5])
    if status != _lib.PEARL_OK:
        rng.consume(draws)
        _lib.check(status, "verify_chain")
    rng.consume(draws)
    return VerifyResult(accepted_count=accepted, correction=None if correction < 0 else correction,
                        examined=examined)


def verify_chain_greedy(drafted: Sequence[TokenId], target_dists: Sequence[ProbDist]) -> VerifyResult:
    """engines._verify_chain_greedy (engines.py:220-226) on the device."""
    n = len(drafted)
    if n == 0:
        return VerifyResult(0, None, 0)
    res, _ = _launch_verify(drafted, [], target_dists, np.zeros(0), _lib.F_GREEDY)
    status, accepted, correction, examined = (int(x) for x in res[:4])
    _lib.check(status, "verify_chain_greedy")
    return VerifyResult(accepted, None if correction < 0 else correction, examined)


def verify_with_bonus(drafted, draft_dists, target_dists, rng: Optional[RandomStream], greedy: bool):
    """SD verify + bonus pick in one launch (engines.py:375-380).

    ``target_dists`` has len(drafted) + 1 rows.  Returns (VerifyResult, bonus).
    """
    n = len(drafted)
    flags = _lib.F_GREEDY if greedy else 0
    us = np.zeros(0) if greedy else rng.peek(n + 2)
    res, _ = _launch_verify(drafted, [] if greedy else draft_dists, target_dists, us, flags)
    status, accepted, correction, examined, draws, bonus = (int(x) for x in res[:6])
    if rng is not None and not greedy:
        rng.consume(draws)
    _lib.check(status, "verify_chain")
    vr = VerifyResult(accepted, None if correction < 0 else correction, examined)
    return vr, (None if bonus < 0 else bonus)
