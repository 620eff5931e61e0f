"""Golden artifacts of the REFERENCE CLI's ``run`` command (pearl_lab.cli,
cli.py:181-277) on synthetic-family run configs: run_summary.json,
summary.csv, outputs.txt, run_hist.csv and every trace_NNN.jsonl.  Run in the
build container (the reference is importable here, not on the GPU box):

    python tests/golden/make_run_golden.py     # writes run_cases.json
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pearl_lab import cli  # noqa: E402  (the reference)

PROMPTS = ["", "hello world", "ab", "PEARL: parallel speculative decoding"]

CASES = [
    {"engine": "pearl", "gamma": 4, "max_new_tokens": 40, "seed": 7, "greedy": False,
     "model": {"synthetic": {"alpha": 0.8, "vocab": 64}}, "timing": {"t": 1.0, "c": 5.0}},
    {"engine": "pearl", "gamma": 2, "max_new_tokens": 33, "seed": 11, "greedy": True,
     "model": {"synthetic": {"alpha": 0.9}}, "timing": {"t": 0.5, "c": 3.0}},
    {"engine": "sd", "gamma": 3, "max_new_tokens": 25, "seed": 3,
     "model": {"synthetic": {"alpha": 0.6, "vocab": 16}}, "timing": {"t": 1.0, "c": 8.0}},
    {"engine": "ar", "max_new_tokens": 12, "seed": 5,
     "model": {"synthetic": {"alpha": 0.5}}, "timing": {"t": 1.0, "c": 2.0}},
    {"engine": "pearl", "gamma": 6, "max_new_tokens": 50, "seed": 1, "no_prompts": True,
     "model": {"synthetic": {"alpha": 0.95, "vocab": 32}}, "timing": {"t": 2.0, "c": 6.0}},
]


def _read(path):
    with open(path, "r", encoding="utf-8") as fh:
        return fh.read()


def main() -> None:
    out = []
    for case in CASES:
        doc = {k: v for k, v in case.items() if k != "no_prompts"}
        with tempfile.TemporaryDirectory() as d:
            if not case.get("no_prompts"):
                with open(os.path.join(d, "prompts.txt"), "w", encoding="utf-8") as fh:
                    fh.write("\n".join(PROMPTS) + "\n")
                doc["prompts"] = os.path.join(d, "prompts.txt")
            with open(os.path.join(d, "cfg.json"), "w") as fh:
                json.dump(doc, fh)
            art = os.path.join(d, "out")
            with contextlib.redirect_stdout(io.StringIO()):
                rc = cli.main(["run", "--config", os.path.join(d, "cfg.json"), "--out", art])
            assert rc == 0, rc
            files = {f: _read(os.path.join(art, f)) for f in sorted(os.listdir(art)) if not f.endswith(".svg")}
        out.append({"config": {k: v for k, v in case.items()}, "files": files})
    with open(os.path.join(HERE, "run_cases.json"), "w") as fh:
        json.dump({"prompts": PROMPTS, "cases": out}, fh, indent=1)
    print(f"{len(out)} run configs recorded")


if __name__ == "__main__":
    main()
