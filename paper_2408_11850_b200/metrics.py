"""Run metrics and trace pricing.

Host-side bookkeeping over the StepTraces every engine returns, so a B200 run
reports what the reference's CLI reports and can be compared with the
reference's discrete-event pricing:

* ``simulate_run`` prices a recorded trace in draft-forward units: a draft
  forward costs t, a target forward costs c*t; AR steps cost c*t, SD steps
  gamma*t + c*t, PEARL steps max(gamma*t, c*t).  The trace itself is never
  re-derived (pearl_lab/simulator.py:34-131).
* ``measured_params`` fills (t, c) from CUDA-event timings of the two GPU
  models, so the simulated speedup can be set next to the measured one.
* ``summarize_run`` aggregates a list of DecodeResults into the CLI's
  RunSummary (cli.py:65-83, 288-315): steps, tokens, tokens per step,
  acceptance, pooled simulated speedup, mean wall time and the draft-run
  histogram (engines.draft_run_lengths, engines.py:176-195).
"""

from __future__ import annotations

import dataclasses
from collections import Counter
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

from .engines import StepTrace, draft_run_lengths


class MismatchedEngine(ValueError):
    """A trace's step kinds do not belong to the claimed engine (simulator.py:29-30)."""


@dataclass(frozen=True)
class TimingParams:
    """Draft forward time t and target/draft cost ratio c, both positive (simulator.py:33-49)."""

    t: float = 1.0
    c: float = 1.0

    def __post_init__(self) -> None:
        if not self.t > 0.0:
            raise ValueError(f"t must be positive, got {self.t}")
        if not self.c > 0.0:
            raise ValueError(f"c must be positive, got {self.c}")

    @property
    def target_time(self) -> float:
        return self.c * self.t


def time_ar_step(params: TimingParams) -> float:
    return params.target_time


def time_sd_step(gamma: int, params: TimingParams) -> float:
    if gamma < 1:
        raise ValueError(f"gamma must be >= 1, got {gamma}")
    return gamma * params.t + params.target_time


def time_pearl_step(gamma: int, params: TimingParams) -> float:
    if gamma < 1:
        raise ValueError(f"gamma must be >= 1, got {gamma}")
    return max(gamma * params.t, params.target_time)


@dataclass(frozen=True)
class SimReport:
    """Timing summary of one simulated run (simulator.py:70-79)."""

    engine: str
    steps: int
    finalized_tokens: int
    total_time: float
    tokens_per_time: float
    speedup_vs_ar: float


_KINDS = {"ar": ("ar",), "sd": ("sd",), "pearl": ("pre_verify", "post_verify")}


def _step_time(kind: str, n_drafted: int, params: TimingParams) -> float:
    if kind == "ar":
        return time_ar_step(params)
    if kind == "sd":
        return time_sd_step(n_drafted, params)
    return time_pearl_step(n_drafted, params)


def simulate_run(steps: Sequence[StepTrace], params: TimingParams, engine_kind: str) -> SimReport:
    """Price a recorded trace under ``params`` (simulator.py:110-131)."""
    if engine_kind not in _KINDS:
        raise MismatchedEngine(f"unknown engine kind {engine_kind!r}")
    if not steps:
        raise MismatchedEngine("empty trace")
    allowed = _KINDS[engine_kind]
    total_time = 0.0
    finalized = 0
    for tr in steps:
        if tr.kind not in allowed:
            raise MismatchedEngine(f"step {tr.index} has kind {tr.kind!r}, not a {engine_kind!r} step")
        total_time += _step_time(tr.kind, len(tr.drafted), params)
        finalized += tr.finalized_delta
    tokens_per_time = finalized / total_time
    return SimReport(engine_kind, len(steps), finalized, total_time, tokens_per_time,
                     tokens_per_time * params.target_time)


def measured_params(target, draft) -> TimingParams:
    """(t, c) of a GPU pair from CUDA-event timed single-token forwards
    (LlamaModel.measure_forward_time): t = draft forward, c = target / draft."""
    t_d = float(draft.measure_forward_time(1))
    t_t = float(target.measure_forward_time(1))
    return TimingParams(t=t_d, c=t_t / t_d)


@dataclass
class RunSummary:
    """Aggregate over all prompts of one run (cli.py:65-83)."""

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
    """cli._aggregate (cli.py:288-315) over DecodeResults: every prompt's
    trace priced with ``params``; the pooled simulated speedup is all
    prompts' tokens repriced against token-at-a-time decoding."""
    kind = "pearl" if engine == "pearl" else engine
    reports = [simulate_run(r.steps, params, kind) for r in results]
    total_steps = sum(rep.steps for rep in reports)
    total_tokens = sum(rep.finalized_tokens for rep in reports)
    total_time = sum(rep.total_time for rep in reports)
    steps = [tr for r in results for tr in r.steps]
    accepted = sum(tr.accepted_count for tr in steps)
    rejected = sum(1 for tr in steps if tr.correction is not None)
    acceptance = accepted / (accepted + rejected) if accepted + rejected else None
    # cli.py:233-237: runs over all prompts' steps back to back (a run still
    # open at the end of one prompt continues into the next); none for AR
    hist = Counter(draft_run_lengths(steps)) if engine != "ar" else Counter()
    walls = [w for w in (walls or []) if w is not None]
    return RunSummary(engine=engine, gamma=gamma, n_prompts=len(results), total_steps=total_steps,
                      total_new_tokens=total_tokens, tokens_per_step=total_tokens / total_steps,
                      acceptance=acceptance, sim_speedup=total_tokens * params.target_time / total_time,
                      mean_wall_seconds=sum(walls) / len(walls) if walls else None,
                      run_length_hist=dict(hist))
