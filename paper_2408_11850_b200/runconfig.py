"""Run configs -> the B200 engines.

The reference decodes a prompt list from a strict JSON "run" config
(``pearl-lab run --config cfg.json``: config.schema.json:38-66,
config.py:81-140, cli.py:181-277).  This module takes the same document and
routes it to this package's engines, writing the same artifacts into
``out_dir``: ``trace_NNN.jsonl`` per prompt, ``summary.csv``, ``outputs.txt``,
``run_hist.csv`` and ``run_summary.json`` (the SVG charts of cli.py are
plotting, not decoding, and are not produced).

Model families:

* ``"synthetic": {"alpha", "vocab"}`` -- the reference's constant-acceptance
  pair (models.make_alpha_pair), decoded through the plugin path; outputs
  equal the reference CLI's (tests/test_runconfig.py against
  tests/golden/run_cases.json).
* ``"transformer": {...}`` (new) -- a GPU Llama pair on the device fast path:
  ``arch`` (a llama.PAIRS name, random-init controlled-alignment weights with
  ``seed``) or ``checkpoint`` ({"target": dir, "draft": dir}, Hugging Face
  safetensors via checkpoint.load_llama), ``dtype`` ("bf16"), ``devices``
  ([target, draft]; one GPU in process -- a draft on another GPU is the split
  pair, split_pair.connect_pair, one process per GPU), ``gemm``,
  ``draft_sms``, ``temperature``, ``eos_id``.  Prompts are token ids: one
  prompt per line of ``prompts`` (whitespace-separated ints; an empty line, or
  no prompts at all, decodes from BOS alone, like the reference's empty
  prompt) or ``synthetic_prompts`` {"n", "length", "seed"}.  ``timing`` is optional and
  measured on the GPU when absent (metrics.measured_params).

Run-level extensions: ``adaptive_gamma``, ``gamma_max`` and ``batch`` (B
prompts decoded in lockstep by batched.py; outputs equal the per-prompt
decodes).  Errors: ``ConfigError`` with the JSON path of the offending field,
exit codes of cli.py:439-452 from ``main``.

    python -m paper_2408_11850_b200.runconfig run --config cfg.json [--out DIR] [--seed S]
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import json
import os
import sys
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np

from .engines import DecodeResult, EngineConfig, write_trace_jsonl
from .errors import DeviceError, InvalidAlpha
from .metrics import TimingParams, simulate_run, summarize_run

SUMMARY_FIELDS = ["prompt", "engine", "gamma", "steps", "new_tokens", "tokens_per_step", "acceptance", "sim_time",
                  "sim_speedup", "wall_seconds"]

_TIMING = {"type": "object", "properties": {"t": {"type": "number", "exclusiveMinimum": 0},
                                            "c": {"type": "number", "exclusiveMinimum": 0}},
           "required": ["t", "c"], "additionalProperties": False}
_SYNTHETIC = {"type": "object", "properties": {"alpha": {"type": "number", "minimum": 0, "maximum": 1},
                                               "vocab": {"type": "integer", "minimum": 2, "default": 64}},
              "required": ["alpha"], "additionalProperties": False}
_TRANSFORMER = {
    "type": "object",
    "properties": {
        "arch": {"type": "string"},
        "checkpoint": {"type": "object", "properties": {"target": {"type": "string"}, "draft": {"type": "string"}},
                       "required": ["target", "draft"], "additionalProperties": False},
        "seed": {"type": "integer"},
        "dtype": {"enum": ["bf16"]},
        "devices": {"type": "array", "items": {"type": "integer", "minimum": 0}, "minItems": 2, "maxItems": 2},
        "gemm": {"enum": ["tcgen05", "cudacore"]},
        "draft_sms": {"type": "integer", "minimum": 0},
        "branch_std": {"type": "number", "exclusiveMinimum": 0},
        "temperature": {"type": "number", "exclusiveMinimum": 0},
        "eos_id": {"type": "integer", "minimum": 0},
    },
    "additionalProperties": False,
}
RUN_SCHEMA = {
    "type": "object",
    "properties": {
        "engine": {"enum": ["ar", "sd", "pearl"]},
        "gamma": {"type": "integer", "minimum": 1},
        "max_new_tokens": {"type": "integer", "minimum": 1},
        "seed": {"type": "integer"},
        "greedy": {"type": "boolean"},
        "prompts": {"type": "string"},
        "synthetic_prompts": {"type": "object",
                              "properties": {"n": {"type": "integer", "minimum": 1},
                                             "length": {"type": "integer", "minimum": 1},
                                             "seed": {"type": "integer"}},
                              "required": ["n", "length", "seed"], "additionalProperties": False},
        "model": {"type": "object", "properties": {"synthetic": _SYNTHETIC, "transformer": _TRANSFORMER},
                  "minProperties": 1, "maxProperties": 1, "additionalProperties": False},
        "timing": _TIMING,
        "adaptive_gamma": {"type": "boolean"},
        "gamma_max": {"type": "integer", "minimum": 1},
        "batch": {"type": "integer", "minimum": 1},
        "out_dir": {"type": "string"},
    },
    "required": ["engine", "max_new_tokens", "seed", "model"],
    "additionalProperties": False,
}


class ConfigError(ValueError):
    """A run config failed validation (config.py:21-31); ``path`` is the JSON
    path of the offending field, e.g. "$.model.transformer.arch"."""

    def __init__(self, path: str, message: str) -> None:
        self.path = path
        super().__init__(f"config error at {path}: {message}")


@dataclass(frozen=True)
class SyntheticSpec:
    alpha: float
    vocab: int = 64


@dataclass(frozen=True)
class TransformerSpec:
    arch: Optional[str] = None
    checkpoint: Optional[Tuple[str, str]] = None  # (target dir, draft dir)
    seed: int = 1234
    dtype: str = "bf16"
    devices: Tuple[int, int] = (0, 0)
    gemm: str = "tcgen05"
    draft_sms: Optional[int] = None
    branch_std: Optional[float] = None
    temperature: float = 1.0
    eos_id: Optional[int] = None


@dataclass(frozen=True)
class RunConfig:
    """A validated run config (config.py:81-94 plus the extensions above)."""

    engine: str
    max_new_tokens: int
    seed: int
    model: Union[SyntheticSpec, TransformerSpec]
    timing: Optional[TimingParams] = None
    gamma: Optional[int] = None
    greedy: bool = False
    prompts: Optional[str] = None
    synthetic_prompts: Optional[Tuple[int, int, int]] = None  # (n, length, seed)
    adaptive_gamma: bool = False
    gamma_max: int = 32
    batch: int = 1
    out_dir: Optional[str] = None


def _validate(doc: dict) -> None:
    import jsonschema
    errors = sorted(jsonschema.Draft202012Validator(RUN_SCHEMA).iter_errors(doc), key=lambda e: e.json_path)
    if errors:
        raise ConfigError(errors[0].json_path, errors[0].message)


def parse_run_config(doc: dict) -> RunConfig:
    """Validate a run document and return the RunConfig (config.py:126-140)."""
    if not isinstance(doc, dict):
        raise ConfigError("$", "top level must be a JSON object")
    _validate(doc)
    engine = doc["engine"]
    if engine in ("sd", "pearl") and "gamma" not in doc:
        raise ConfigError("$.gamma", f"engine {engine!r} requires gamma")
    if doc.get("batch", 1) > 1 and doc.get("adaptive_gamma", False):
        raise ConfigError("$.adaptive_gamma", "batched (lockstep) decoding drafts a fixed gamma")
    if "prompts" in doc and "synthetic_prompts" in doc:
        raise ConfigError("$.synthetic_prompts", "give either prompts or synthetic_prompts")
    timing = TimingParams(t=doc["timing"]["t"], c=doc["timing"]["c"]) if "timing" in doc else None
    if "synthetic" in doc["model"]:
        m = doc["model"]["synthetic"]
        model: Union[SyntheticSpec, TransformerSpec] = SyntheticSpec(alpha=m["alpha"], vocab=m.get("vocab", 64))
        if timing is None:
            raise ConfigError("$.timing", "required for the synthetic model family")
        if "synthetic_prompts" in doc:
            raise ConfigError("$.synthetic_prompts", "token-id prompts need the transformer model family")
    else:
        m = doc["model"]["transformer"]
        from .llama import PAIRS
        if ("arch" in m) == ("checkpoint" in m):
            raise ConfigError("$.model.transformer", "give exactly one of arch and checkpoint")
        if "arch" in m and m["arch"] not in PAIRS:
            raise ConfigError("$.model.transformer.arch", f"{m['arch']!r} is not one of {sorted(PAIRS)}")
        devices = tuple(m.get("devices", (0, 0)))
        if devices[0] != devices[1]:
            raise ConfigError("$.model.transformer.devices",
                              "a draft on another GPU runs as a split pair, one process per GPU "
                              "(split_pair.connect_pair); an in-process run takes one device")
        ck = m.get("checkpoint")
        model = TransformerSpec(arch=m.get("arch"), checkpoint=(ck["target"], ck["draft"]) if ck else None,
                                seed=m.get("seed", 1234), dtype=m.get("dtype", "bf16"), devices=devices,
                                gemm=m.get("gemm", "tcgen05"), draft_sms=m.get("draft_sms"),
                                branch_std=m.get("branch_std"), temperature=m.get("temperature", 1.0),
                                eos_id=m.get("eos_id"))
    sp = doc.get("synthetic_prompts")
    return RunConfig(engine=engine, max_new_tokens=doc["max_new_tokens"], seed=doc["seed"], model=model,
                     timing=timing, gamma=doc.get("gamma"), greedy=doc.get("greedy", False),
                     prompts=doc.get("prompts"), synthetic_prompts=(sp["n"], sp["length"], sp["seed"]) if sp else None,
                     adaptive_gamma=doc.get("adaptive_gamma", False), gamma_max=doc.get("gamma_max", 32),
                     batch=doc.get("batch", 1), out_dir=doc.get("out_dir"))


def load_run_config(path: str) -> RunConfig:
    """Read and validate a run config file (config.py:36-48, 126-140)."""
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ConfigError("$", f"not valid JSON: {exc}") from exc
    return parse_run_config(doc)


def derive_seed(seed: int, index: int) -> int:
    """Per-prompt seed (cli.py:94-96)."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(index,))
    return int(ss.generate_state(1, np.uint64)[0])


def build_models(cfg: RunConfig, max_seq: int = 1024):
    """(draft, target, eos_id, timing) for a run config (cli.py:99-121)."""
    if isinstance(cfg.model, SyntheticSpec):
        from .models import make_alpha_pair
        pair = make_alpha_pair(cfg.model.alpha, cfg.model.vocab, draft_time=cfg.timing.t,
                               target_time=cfg.timing.target_time)
        return pair.draft, pair.target, None, cfg.timing
    import torch
    from . import llama
    spec = cfg.model
    torch.cuda.set_device(spec.devices[0])
    max_tokens = 128 if spec.gemm == "tcgen05" else 64
    eos_id = spec.eos_id
    if spec.checkpoint is not None:
        from .checkpoint import load_llama
        if spec.branch_std is not None:
            raise ConfigError("$.model.transformer.branch_std", "applies to random-init arch pairs, not checkpoints")
        try:
            tc, tw = load_llama(spec.checkpoint[0], device="cuda")
            dc, dw = load_llama(spec.checkpoint[1], device="cuda")
        except ValueError as exc:
            raise ConfigError("$.model.transformer.checkpoint", str(exc)) from exc
        if tc.vocab != dc.vocab:
            raise ConfigError("$.model.transformer.checkpoint", f"vocab mismatch: target {tc.vocab}, draft {dc.vocab}")
        if tc.bos_id != dc.bos_id:
            raise ConfigError("$.model.transformer.checkpoint", f"bos mismatch: target {tc.bos_id}, draft {dc.bos_id}")
        target, draft = llama.pair_from_weights(tc, tw, dc, dw, gemm_target=spec.gemm, max_seq=max_seq,
                                                max_tokens=max_tokens, temperature=spec.temperature,
                                                n_slots=cfg.batch, draft_sms=spec.draft_sms or 0)
        if eos_id is None:
            eos_id = tc.eos_id  # config.json's eos_token_id
    else:
        align = llama.AlignSpec(seed=spec.seed, branch_std=spec.branch_std if spec.branch_std is not None
                                else llama.PAIR_BRANCH_STD[spec.arch])
        target, draft = llama.build_pair(spec.arch, gemm_target=spec.gemm, align=align, max_seq=max_seq,
                                         max_tokens=max_tokens, temperature=spec.temperature, n_slots=cfg.batch,
                                         draft_sms=spec.draft_sms if spec.draft_sms is not None
                                         else llama.PAIR_DRAFT_SMS[spec.arch])
    timing = cfg.timing
    if timing is None:
        from .metrics import measured_params
        timing = measured_params(target, draft)
    return draft, target, eos_id, timing


def load_prompts(cfg: RunConfig, vocab: Optional[int] = None) -> List[List[int]]:
    """Prompt token lists: text lines -> UTF-8 bytes for the synthetic family
    (cli.py:124-128, textdata.encode_text); whitespace-separated ids (checked
    against ``vocab`` when given) or seeded uniform ids (bench.py's prompts)
    for the transformer family."""
    if cfg.synthetic_prompts is not None:
        n, length, seed = cfg.synthetic_prompts
        if vocab is None:
            return [[0] * length for _ in range(n)]  # lengths only (sizing the KV cache)
        rng = np.random.default_rng(seed)
        return [rng.integers(2, vocab, length).tolist() for _ in range(n)]
    if cfg.prompts is None:
        lines = [""]
    else:
        with open(cfg.prompts, "r", encoding="utf-8") as fh:
            lines = fh.read().splitlines() or [""]
    if isinstance(cfg.model, SyntheticSpec):
        return [list(line.encode("utf-8")) for line in lines]
    out = []
    for i, line in enumerate(lines):
        try:
            ids = [int(x) for x in line.split()]
        except ValueError as exc:
            raise ConfigError("$.prompts", f"line {i + 1}: token ids must be integers ({exc})") from exc
        if vocab is not None and any(not 0 <= t < vocab for t in ids):
            raise ConfigError("$.prompts", f"line {i + 1}: token ids must be in [0, {vocab})")
        out.append(ids)
    return out


def _decode_all(cfg: RunConfig, draft, target, prompts, eos_id, real_latency: bool):
    """DecodeResults and wall seconds per prompt, per-prompt derived seeds."""
    gamma = cfg.gamma if cfg.gamma is not None else 1
    temp = cfg.model.temperature if isinstance(cfg.model, TransformerSpec) else 1.0
    device = isinstance(cfg.model, TransformerSpec)
    ecfgs = [EngineConfig(gamma=gamma, max_new_tokens=cfg.max_new_tokens, seed=derive_seed(cfg.seed, i),
                          greedy=cfg.greedy, eos_id=eos_id, real_latency=real_latency, temperature=temp,
                          adaptive_gamma=cfg.adaptive_gamma, gamma_max=max(cfg.gamma_max, gamma))
             for i in range(len(prompts))]
    results: List[DecodeResult] = []
    walls: List[Optional[float]] = []
    if device and cfg.batch > 1:
        from . import batched
        fn = {"pearl": batched.decode_pearl_batch, "sd": batched.decode_sd_batch}.get(cfg.engine)
        for lo in range(0, len(prompts), cfg.batch):
            chunk = prompts[lo:lo + cfg.batch]
            seeds = [e.seed for e in ecfgs[lo:lo + cfg.batch]]
            t0 = time.perf_counter()
            if fn is None:
                got = batched.decode_autoregressive_batch(target, chunk, ecfgs[0], seeds=seeds)
            else:
                got = fn(draft, target, chunk, ecfgs[0], seeds=seeds)
            wall = time.perf_counter() - t0
            results.extend(got)
            walls.extend([wall] * len(got))
        return results, walls
    from . import engines
    for p, ecfg in zip(prompts, ecfgs):
        t0 = time.perf_counter()
        if cfg.engine == "ar":
            r = engines.decode_autoregressive(target, p, ecfg)
        elif cfg.engine == "sd":
            r = engines.decode_sd(draft, target, p, ecfg)
        else:
            r = engines.decode_pearl(draft, target, p, ecfg)
        walls.append(time.perf_counter() - t0 if (device or real_latency) else None)
        results.append(r)
    return results, walls


def _acceptance(result: DecodeResult) -> Optional[float]:
    accepted = sum(tr.accepted_count for tr in result.steps)
    rejected = sum(1 for tr in result.steps if tr.correction is not None)
    return accepted / (accepted + rejected) if accepted + rejected else None


def run(cfg: RunConfig, out_dir: Optional[str] = None, real_latency: bool = False, models=None):
    """Decode every prompt of ``cfg`` and write cli.py's run artifacts
    (cli.py:181-277).  ``models``: prebuilt (draft, target, eos_id, timing)
    to reuse across runs.  Returns the RunSummary."""
    out_dir = out_dir or cfg.out_dir
    if out_dir is None:
        raise ConfigError("$.out_dir", "missing; set it in the config or pass --out")
    os.makedirs(out_dir, exist_ok=True)
    if models is None:
        max_seq = 1024
        if isinstance(cfg.model, TransformerSpec):
            longest = max(len(p) for p in load_prompts(cfg)) + 1  # + BOS
            max_seq = longest + cfg.max_new_tokens + 2 * max(cfg.gamma or 1, cfg.gamma_max) + 16
            if max_seq > 4096:
                raise ConfigError("$.prompts", f"longest prompt + max_new_tokens + draft slack needs a KV cache of "
                                  f"{max_seq} positions; the kernels hold at most 4096")
        models = build_models(cfg, max_seq=max_seq)
    draft, target, eos_id, timing = models
    prompts = load_prompts(cfg, target.vocab_size)
    gamma = cfg.gamma if cfg.gamma is not None else 1
    results, walls = _decode_all(cfg, draft, target, prompts, eos_id, real_latency)
    reports = [simulate_run(r.steps, timing, cfg.engine) for r in results]

    for i, r in enumerate(results):
        write_trace_jsonl(r.steps, os.path.join(out_dir, f"trace_{i:03d}.jsonl"))
    with open(os.path.join(out_dir, "summary.csv"), "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(SUMMARY_FIELDS)
        for i, (r, rep, wall) in enumerate(zip(results, reports, walls)):
            acc = _acceptance(r)
            w.writerow([i, cfg.engine, gamma, rep.steps, rep.finalized_tokens,
                        f"{rep.finalized_tokens / rep.steps:.6f}", "" if acc is None else f"{acc:.6f}",
                        f"{rep.total_time:.6f}", f"{rep.speedup_vs_ar:.6f}", "" if wall is None else f"{wall:.6f}"])
    with open(os.path.join(out_dir, "outputs.txt"), "w", encoding="utf-8") as fh:
        for r in results:
            fh.write(" ".join(str(t) for t in r.tokens) + "\n")
    summary = summarize_run(cfg.engine, gamma, results, timing, walls)
    if summary.run_length_hist:
        top = max(summary.run_length_hist)
        with open(os.path.join(out_dir, "run_hist.csv"), "w", encoding="utf-8", newline="") as fh:
            fh.write("run_length,count\n")
            for k in range(top + 1):
                fh.write(f"{k},{summary.run_length_hist.get(k, 0)}\n")
    with open(os.path.join(out_dir, "run_summary.json"), "w", encoding="utf-8") as fh:
        json.dump(summary.to_dict(), fh, indent=2)
        fh.write("\n")
    return summary


def main(argv: Optional[Sequence[str]] = None) -> int:
    """``run`` subcommand of cli.py:381-395; exit codes 0 / 2 (config) / 3 (I/O)."""
    ap = argparse.ArgumentParser(prog="paper_2408_11850_b200.runconfig")
    sub = ap.add_subparsers(dest="command", required=True)
    r = sub.add_parser("run", help="decode prompts with one engine and emit artifacts")
    r.add_argument("--config", required=True)
    r.add_argument("--seed", type=int, default=None)
    r.add_argument("--out", default=None)
    r.add_argument("--real-latency", action="store_true")
    args = ap.parse_args(argv)
    try:
        cfg = load_run_config(args.config)
        if args.seed is not None:
            cfg = dataclasses.replace(cfg, seed=args.seed)
        s = run(cfg, args.out, real_latency=args.real_latency)
    except (ConfigError, InvalidAlpha) as exc:
        print(f"pearl-b200: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"pearl-b200: {exc}", file=sys.stderr)
        return 3
    except (DeviceError, ValueError) as exc:
        print(f"pearl-b200: {exc}", file=sys.stderr)
        return 2
    print(f"{s.engine}: {s.total_new_tokens} tokens over {s.n_prompts} prompts, "
          f"{s.tokens_per_step:.3f} tokens/step, sim speedup {s.sim_speedup:.3f}")
    print(f"artifacts in {args.out or cfg.out_dir}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
