"""Run metrics and trace pricing.

Host-side bookkeeping over the StepTraces every engine returns, so a B200 run
reports the quantities the reference's CLI reports (cli.py:65-83, 288-315)
and can be set next to the reference's discrete-event pricing
(simulator.py:110-131).

Pricing model (the reference's definition, in draft-forward units): a draft
forward costs t and a target forward c·t.  A step that drafted g tokens costs

    serial phases   (AR, SD)             draft_part + target_part
    overlapped      (PEARL pre / post)   max(draft_part, target_part)

with draft_part = g·t (0 for AR) and target_part = c·t.  Here a trace is
first turned into arrays (kind code, drafted count, finalized count) and
priced in one vectorised pass; the total is the sequential (left-to-right)
sum of the step costs, which is what the reference accumulates, so the
priced totals are bit-identical to it (tests/test_metrics_cpu.py pins them
to pearl_lab.simulator outputs on the reference's own traces).

``measured_params`` fills (t, c) from CUDA-event timings of the two GPU
models, so the simulated speedup can be compared with the measured one.
"""

from __future__ import annotations

import dataclasses
from collections import Counter
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

from .engines import StepTrace, draft_run_lengths


class MismatchedEngine(ValueError):
    """A trace's step kinds do not belong to the claimed engine (simulator.py:29-30)."""


@dataclass(frozen=True)
class TimingParams:
    """Draft forward time ``t`` and target/draft cost ratio ``c``, both > 0."""

    t: float = 1.0
    c: float = 1.0

    def __post_init__(self) -> None:
        for name in ("t", "c"):
            if not getattr(self, name) > 0.0:
                raise ValueError(f"{name} must be positive, got {getattr(self, name)}")

    @property
    def target_time(self) -> float:
        return self.c * self.t


@dataclass(frozen=True)
class SimReport:
    """Priced totals of one trace (simulator.py:70-79)."""

    engine: str
    steps: int
    finalized_tokens: int
    total_time: float
    tokens_per_time: float
    speedup_vs_ar: float


# step kind -> (code, drafts, overlapped); the engine kinds each accept a set of codes
_STEP_KINDS = {"ar": (0, False, False), "sd": (1, True, False),
               "pre_verify": (2, True, True), "post_verify": (3, True, True)}
_ENGINE_CODES = {"ar": {0}, "sd": {1}, "pearl": {2, 3}}


def _trace_arrays(steps: Sequence[StepTrace], engine_kind: str):
    """(drafted counts, overlapped flags, drafting flags, finalized counts),
    validating every step's kind against the engine."""
    if engine_kind not in _ENGINE_CODES:
        raise MismatchedEngine(f"unknown engine kind {engine_kind!r}")
    if not steps:
        raise MismatchedEngine("empty trace")
    ok = _ENGINE_CODES[engine_kind]
    n = len(steps)
    g = np.empty(n, np.float64)
    overlap = np.empty(n, bool)
    drafts = np.empty(n, bool)
    fin = np.empty(n, np.int64)
    for i, tr in enumerate(steps):
        spec = _STEP_KINDS.get(tr.kind)
        if spec is None or spec[0] not in ok:
            raise MismatchedEngine(f"step {tr.index} has kind {tr.kind!r}, not a {engine_kind!r} step")
        g[i], drafts[i], overlap[i], fin[i] = len(tr.drafted), spec[1], spec[2], tr.finalized_delta
    if np.any(drafts & (g < 1)):
        raise ValueError("gamma must be >= 1 for a drafting step")
    return g, overlap, drafts, fin


def step_costs(steps: Sequence[StepTrace], params: TimingParams, engine_kind: str) -> np.ndarray:
    """Per-step cost of a trace under ``params`` (see the module doc)."""
    g, overlap, drafts, _ = _trace_arrays(steps, engine_kind)
    draft_part = np.where(drafts, g * params.t, 0.0)
    target_part = np.full_like(g, params.target_time)
    return np.where(overlap, np.maximum(draft_part, target_part),
                    np.where(drafts, draft_part + target_part, target_part))


def simulate_run(steps: Sequence[StepTrace], params: TimingParams, engine_kind: str) -> SimReport:
    """Price a recorded trace (simulator.py:110-131); the trace is never re-derived."""
    costs = step_costs(steps, params, engine_kind)
    total = float(np.cumsum(costs)[-1])  # sequential, as the reference accumulates
    finalized = int(sum(tr.finalized_delta for tr in steps))
    rate = finalized / total
    return SimReport(engine_kind, len(steps), finalized, total, rate, rate * params.target_time)


def measured_params(target, draft) -> TimingParams:
    """(t, c) of a GPU pair from CUDA-event timed single-token forwards
    (LlamaModel.measure_forward_time): t = draft forward, c = target / draft."""
    t_d = float(draft.measure_forward_time(1))
    return TimingParams(t=t_d, c=float(target.measure_forward_time(1)) / t_d)


@dataclass
class RunSummary:
    """Aggregate over all prompts of one run; field names and order are the
    reference CLI's run_summary.json schema (cli.py:65-83)."""

    engine: str
    gamma: int
    n_prompts: int
    total_steps: int
    total_new_tokens: int
    tokens_per_step: float
    acceptance: Optional[float]
    sim_speedup: float
    mean_wall_seconds: Optional[float]
    run_length_hist: Dict[int, int]

    def to_dict(self) -> dict:
        d = dataclasses.asdict(self)
        d["run_length_hist"] = {str(k): v for k, v in sorted(self.run_length_hist.items())}
        return d


def summarize_run(engine: str, gamma: int, results: Sequence, params: TimingParams,
                  walls: Optional[Sequence[float]] = None) -> RunSummary:
    """One RunSummary over DecodeResults: every prompt's trace priced with
    ``params``; the pooled simulated speedup reprices all prompts' tokens
    against token-at-a-time decoding (N·c·t for N tokens)."""
    reports = [simulate_run(r.steps, params, engine) for r in results]
    steps = [tr for r in results for tr in r.steps]
    n_steps = sum(rep.steps for rep in reports)
    n_tokens = sum(rep.finalized_tokens for rep in reports)
    priced = sum(rep.total_time for rep in reports)
    accepted = sum(tr.accepted_count for tr in steps)
    rejects = sum(tr.correction is not None for tr in steps)
    # draft runs span all prompts' steps back to back (cli.py:233-237); AR has none
    hist = dict(Counter(draft_run_lengths(steps))) if engine != "ar" else {}
    w = [x for x in (walls or ()) if x is not None]
    return RunSummary(engine=engine, gamma=gamma, n_prompts=len(results), total_steps=n_steps,
                      total_new_tokens=n_tokens, tokens_per_step=n_tokens / n_steps,
                      acceptance=accepted / (accepted + rejects) if accepted + rejects else None,
                      sim_speedup=n_tokens * params.target_time / priced,
                      mean_wall_seconds=sum(w) / len(w) if w else None, run_length_hist=hist)
