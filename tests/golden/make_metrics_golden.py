"""Golden outputs of the REFERENCE trace pricing (pearl_lab.simulator) and
run-length accounting (pearl_lab.engines.draft_run_lengths) over the committed
reference engine traces (engine_traces.json).  Run in the build container:

    python tests/golden/make_metrics_golden.py     # writes metrics_cases.json
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pearl_lab.engines import StepTrace, draft_run_lengths  # noqa: E402  (the reference)
from pearl_lab.simulator import TimingParams, simulate_run  # noqa: E402

PARAMS = [(1.0, 1.0), (0.25, 4.0), (1.0, 35.0), (3.4e-3, 7.2)]


def _trace(steps):
    return [StepTrace(s["step"], s["kind"], tuple(s["drafted"]), s["accepted_count"], s["correction"],
                      s["finalized_delta"], s["draft_time"], s["target_time"]) for s in steps]


def main() -> None:
    cases = json.load(open(os.path.join(HERE, "engine_traces.json")))
    out = []
    for ci, case in enumerate(cases):
        for engine in ("ar", "sd", "pearl"):
            if engine not in case:
                continue
            steps = _trace(case[engine]["steps"])
            if not steps:
                continue
            sims = []
            for t, c in PARAMS:
                r = simulate_run(steps, TimingParams(t=t, c=c), engine)
                sims.append({"t": t, "c": c, "steps": r.steps, "finalized": r.finalized_tokens,
                             "total_time": r.total_time, "tokens_per_time": r.tokens_per_time,
                             "speedup_vs_ar": r.speedup_vs_ar})
            out.append({"case": ci, "engine": engine, "sims": sims, "run_lengths": draft_run_lengths(steps)})
    json.dump(out, open(os.path.join(HERE, "metrics_cases.json"), "w"))
    print(f"{len(out)} traces priced")


if __name__ == "__main__":
    main()
