"""CPU: trace pricing and run summaries (metrics.py) against the
reference simulator's outputs on the reference's own engine traces
(tests/golden/metrics_cases.json, made by make_metrics_golden.py)."""

import math

import pytest

from conftest import load_golden


def _steps(raw):
    from paper_2408_11850_b200.engines import StepTrace
    return [StepTrace(s["step"], s["kind"], tuple(s["drafted"]), s["accepted_count"], s["correction"],
                      s["finalized_delta"], s["draft_time"], s["target_time"]) for s in raw]


def test_simulate_run_and_run_lengths_match_reference():
    from paper_2408_11850_b200 import metrics
    from paper_2408_11850_b200.engines import draft_run_lengths
    traces = load_golden("engine_traces.json")
    cases = load_golden("metrics_cases.json")
    assert len(cases) > 50
    for case in cases:
        steps = _steps(traces[case["case"]][case["engine"]]["steps"])
        assert draft_run_lengths(steps) == case["run_lengths"]
        for sim in case["sims"]:
            r = metrics.simulate_run(steps, metrics.TimingParams(t=sim["t"], c=sim["c"]), case["engine"])
            assert (r.steps, r.finalized_tokens) == (sim["steps"], sim["finalized"])
            assert r.total_time == sim["total_time"] and r.tokens_per_time == sim["tokens_per_time"]
            assert r.speedup_vs_ar == sim["speedup_vs_ar"]


def test_simulate_run_errors():
    from paper_2408_11850_b200 import metrics
    traces = load_golden("engine_traces.json")
    steps = _steps(traces[0]["pearl"]["steps"])
    with pytest.raises(metrics.MismatchedEngine):
        metrics.simulate_run(steps, metrics.TimingParams(), "sd")
    with pytest.raises(metrics.MismatchedEngine):
        metrics.simulate_run([], metrics.TimingParams(), "ar")
    with pytest.raises(ValueError):
        metrics.TimingParams(t=0.0)


def test_summarize_run_pools_prompts():
    from paper_2408_11850_b200 import metrics
    from paper_2408_11850_b200.engines import DecodeResult
    traces = load_golden("engine_traces.json")
    res = [DecodeResult(tuple(c["pearl"]["tokens"]), tuple(_steps(c["pearl"]["steps"]))) for c in traces[:6]]
    p = metrics.TimingParams(t=1.0, c=4.0)
    s = metrics.summarize_run("pearl", 4, res, p, walls=[1.0, 3.0])
    reps = [metrics.simulate_run(r.steps, p, "pearl") for r in res]
    assert s.total_steps == sum(r.steps for r in reps)
    assert s.total_new_tokens == sum(r.finalized_tokens for r in reps)
    assert math.isclose(s.sim_speedup, s.total_new_tokens * 4.0 / sum(r.total_time for r in reps))
    assert s.mean_wall_seconds == 2.0 and s.n_prompts == 6
    assert sum(s.run_length_hist.values()) == sum(1 for r in res for st in r.steps if st.correction is not None)
    assert set(s.to_dict()["run_length_hist"]) <= {str(k) for k in s.run_length_hist}
