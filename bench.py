"""Benchmark: PEARL decoding on B200 (BASELINE.json metric, configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (configs[1] of BASELINE.json): Llama-2-7B target + Llama-68M draft,
random-init bf16 weights (controlled-alignment init, llama.py), batch 1,
synthetic 128-token prompts, 128 new tokens.  A *step* is one
``decode_pearl`` call (prefill + decode of 128 tokens) through the public
API.  AR and vanilla SD run on the same kernels in the same process.

N = 1: draft and target co-resident on one B200.  PEARL (the headline) uses
the adaptive draft length with a FROZEN planner calibration
(profiles/planner_calib_*.json, so its gamma schedule depends on the tokens
only) and its concurrent draft on a green-context SM partition; AR and SD
run their target on the whole GPU.  Reported beside it: AR, SD at each
fixed gamma (speedup_vs_sd divides by the BEST one), fixed-gamma PEARL, the
gamma histogram, the per-decode spread and a T=0 leg.

N >= 2 (torchrun): N/2 split pairs -- target on GPU 2i, draft on GPU 2i+1,
one K6 draft->target exchange per step (split_pair.py) -- each decoding its
own prompt shard; value = all pairs' tokens / max-over-ranks time
(``--replicas``: co-resident replicas per GPU instead).

Metric: generated tokens/s (whole job, all ranks), plus speedup vs AR and
vs vanilla SD and mean accepted tokens per target forward.
  value = tokens / device time of the decode graphs (inputs resident)
  e2e   = tokens / wall time of the public API calls (host prompt in, host
          tokens out: H2D of prompt + uniform tables, D2H of step summaries)
Weights (13.6 GB) exceed L2 (126 MB), so every forward streams from HBM.

--impl reference: the reference algorithm's CPU path (oracle/ port of
pearl_lab's decode_pearl driving a PyTorch CPU Llama of the same
architecture) timed on the host cores over a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2408_11850_b200.llama import PAIR_BRANCH_STD, PAIR_DRAFT_SMS  # noqa: E402  (calibration notes there)

METRIC = "tokens/sec & speedup vs AR and vanilla SD; mean accepted tokens/target fwd"
UNIT = "tokens/s"


def _peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _traffic():
    p = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _prompts(n, P, V, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(2, V, P).tolist() for _ in range(n)]


def _calib_path(pair, temp):
    slug = pair.replace("/", "_")
    return os.path.join(REPO, "profiles", f"planner_calib_{slug}_T{'0' if temp is None else f'{temp:g}'}.json")


def planner_calibration(draft, target, args, prompt, greedy, temp):
    """Frozen planner table (fastpath.PlannerCalibration): the committed one
    for this pair (profiles/planner_calib_*.json, measured on B200) unless
    --live-calibration; measured here otherwise and written to gpurun_out/.
    Installed before any timed decode, so the adaptive gamma schedule is a
    function of the decode's tokens only (reproducible across boxes)."""
    from paper_2408_11850_b200 import fastpath
    path = _calib_path(args.pair, 0.0 if greedy else temp)
    if os.path.exists(path) and not args.live_calibration:
        with open(path) as fh:
            cal = fastpath.PlannerCalibration.from_json(json.load(fh), source=os.path.relpath(path, REPO))
    else:
        cal = fastpath.calibrate_planner(draft, target, prompt, args.gamma_max, temperature=temp, greedy=greedy,
                                         new_tokens=min(96, args.new))
        os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
        with open(os.path.join(REPO, "gpurun_out", os.path.basename(path)), "w") as fh:
            json.dump(cal.to_json(), fh, indent=1)
    fastpath.set_planner_calibration(draft, target, cal)
    return cal


def _leg_stats(res, kind, pk):
    steps = [st for r in res for st in r.steps]
    toks = [len(r.tokens) for r in res]
    dev = [r.stats["device_s"] for r in res]
    out = dict(tokens=sum(toks), device_s=sum(dev),
               launches=sum(r.stats["launches"] for r in res),
               replays=sum(r.stats.get("replays", 0) for r in res),
               mean_tok_per_fwd=pk.mean_tokens_per_target_forward(steps),
               alpha=pk.empirical_acceptance(steps) if kind != "ar" else None,
               fallbacks=sum(r.stats.get("fallbacks", 0) for r in res),
               per_decode=[t / d for t, d in zip(toks, dev) if d > 0])
    gs = [g for r in res for g in r.stats.get("gammas", [])]
    if gs:
        hist = {}
        for g in gs:
            hist[str(g)] = hist.get(str(g), 0) + 1
        out["gamma_hist"] = dict(sorted(hist.items(), key=lambda kv: int(kv[0])))
    return out


def _spread(v):
    if not v:
        return None
    return {"min": round(min(v), 2), "median": round(statistics.median(v), 2), "max": round(max(v), 2)}


def run_gpu(args):
    """N = 1 (and --replicas): draft and target co-resident on each GPU."""
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    # PEARL_BENCH_BACKEND=gloo + fewer GPUs than ranks: a functional run of the
    # N>1 path on a 1-GPU box (ranks share cuda:0; the numbers mean nothing)
    backend = os.environ.get("PEARL_BENCH_BACKEND", "nccl")
    if ws > 1:
        dist.init_process_group(backend, init_method="env://")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if ws >= 2 and ws % 2 == 0 and not args.replicas:
        return run_split(args, ws, rank, local)
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import llama

    align = llama.AlignSpec(branch_std=args.branch_std if args.branch_std is not None else PAIR_BRANCH_STD[args.pair],
                            kappa=args.kappa)
    sweep_bs = [int(b) for b in args.batch_sweep.split(",") if b] if args.batch_sweep else []
    greedy = args.temperature <= 0
    temp = 1.0 if greedy else args.temperature
    max_seq = args.prompt + args.new + 2 * args.gamma_max + 16
    target, draft = llama.build_pair(args.pair, gemm_target=args.gemm_target, align=align, max_seq=max_seq,
                                     max_tokens=128, temperature=temp, n_slots=max([1] + sweep_bs),
                                     draft_sms=args.draft_sms if args.draft_sms is not None
                                     else int(os.environ.get("PEARL_DRAFT_SMS", PAIR_DRAFT_SMS[args.pair])))
    # AR and SD never overlap two models: they run on the target over the
    # WHOLE GPU (its own stream-K grids), not on PEARL's partition
    target_full = target.clone(sm_count=0) if getattr(target, "green_partition", None) is not None else target
    # likewise SD's draft: a tcgen05 draft built for PEARL's partition sizes its
    # stream-K grids to it; SD runs it alone on the whole GPU (a CUDA-core draft's
    # grids do not depend on the SM count)
    draft_full = (draft.clone(sm_count=0)
                  if getattr(target, "green_partition", None) is not None and draft.gemm == "tcgen05" else draft)
    V = target.cfg.vocab
    draft_sms_used = getattr(target, "green_partition", (None, None, 0, 0))[2]
    prompts = _prompts(args.warmup + args.steps, args.prompt, V, seed=1000 + rank)

    def cfg_for(gamma, seed, adaptive=False, g=greedy):
        return pk.EngineConfig(gamma=gamma, max_new_tokens=args.new, seed=seed, greedy=g, temperature=temp,
                               adaptive_gamma=adaptive, gamma_max=args.gamma_max)

    cal = planner_calibration(draft, target, args, prompts[0], greedy, temp)
    sd_gammas = [int(g) for g in args.sd_gammas.split(",")]
    pearl_fixed = [int(g) for g in args.pearl_gammas.split(",") if g]

    def run(kind, i, g=greedy):
        seed = 17 + i
        if kind == "pearl":
            return pk.decode_pearl(draft, target, prompts[i], cfg_for(args.gamma, seed, True, g))
        if kind.startswith("pearl"):
            return pk.decode_pearl(draft, target, prompts[i], cfg_for(int(kind[5:]), seed, False, g))
        if kind.startswith("sd"):
            return pk.decode_sd(draft_full, target_full, prompts[i], cfg_for(int(kind[2:]), seed, False, g))
        return pk.decode_autoregressive(target_full, prompts[i], cfg_for(1, seed, False, g))

    def leg(kind, g=greedy, clocks=False):
        for i in range(args.warmup):
            run(kind, i, g)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        ck = Clocks(local) if clocks else None
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        res = [run(kind, args.warmup + i, g) for i in range(args.steps)]
        ev1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = _leg_stats(res, kind, pk)
        st.update(wall_s=wall, event_s=ev0.elapsed_time(ev1) / 1e3)
        if ws > 1:
            dist.barrier()
        return st, res, (ck.stop() if ck else None)

    results, timed = {}, {}
    kinds = ["ar"] + [f"sd{g}" for g in sd_gammas] + [f"pearl{g}" for g in pearl_fixed] + ["pearl"]
    clocks = None
    for kind in kinds:  # adaptive PEARL (the headline) last: its clocks are sampled
        results[kind], timed[kind], ck = leg(kind, clocks=kind == "pearl")
        clocks = ck or clocks
    greedy_leg = None
    if args.greedy_leg and not greedy:
        # BASELINE configs[1]: temperature 0 as well (greedy device path), with
        # the pair's T=0 planner table (committed, or measured under
        # --live-calibration): alpha-hat 1 prices long draft blocks differently
        planner_calibration(draft, target, args, prompts[0], True, temp)
        g_res = {}
        for kind in ["ar"] + [f"sd{g}" for g in sd_gammas] + ["pearl"]:
            g_res[kind] = leg(kind, g=True)[0]
        greedy_leg = summarize_legs(g_res, ws, sd_gammas, [])
    agg = {k: aggregate_one(v, ws) for k, v in results.items()}
    # dominant kernel sequence: the target window forward at the adaptive
    # decodes' most frequent draft length (their post-verify window)
    hist = results["pearl"].get("gamma_hist", {str(args.gamma): 1})
    g_mode = int(max(hist.items(), key=lambda kv: kv[1])[0])
    rl = roofline(target, draft, g_mode, args)
    rl["by_window"] = {str(m): window_frac(target, m, args) for m in sorted({1, 4, g_mode, 16})}
    summary = run_summaries(target, draft, timed, args)
    split_model = split_pair_model(target, draft, results["pearl"]["alpha"]) if ws == 1 else None
    target_bytes, draft_bytes = target.cfg.weight_bytes(), draft.cfg.weight_bytes()
    sweep = batch_sweep(target_full, draft_full, args, sweep_bs, greedy, temp, ws) if sweep_bs else None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(target, draft, prompts[0], args, greedy, temp)
    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return None
    legs = summarize_legs(results, ws, sd_gammas, pearl_fixed, agg)
    wbytes = target_bytes + draft_bytes
    dp, ep, wp, tp = agg["pearl"]
    line = {
        "metric": METRIC,
        "value": round(tp / dp, 2),
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * ep / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic prompts (uniform random ids), random-init weights (controlled-alignment init)",
        "config": {
            "workload": f"{args.pair} PEARL (adaptive draft length), batch 1, prompt {args.prompt}, "
                        f"{args.new} new tokens, {'greedy T=0' if greedy else f'T={temp:g}'}, "
                        f"draft+target co-resident per GPU",
            "pair": args.pair, "global_batch": ws, "prompt_len": args.prompt, "new_tokens": args.new,
            "adaptive_gamma": True, "gamma_max": args.gamma_max,
            "planner_calibration": cal.source, "temperature": 0.0 if greedy else temp,
            "target_gemm": args.gemm_target, "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
            "draft_sms": draft_sms_used, "ar_sd_target": "whole GPU (own stream-K grids, target and tcgen05 draft)",
            "l2": f"weights {wbytes / 1e9:.2f} GB vs 126 MB L2: "
                  + ("every forward streams HBM (no flush needed)" if wbytes > 126e6 else "L2-resident (tiny pair)"),
        },
        "e2e": {"value": round(tp / wp, 2), "unit": UNIT,
                # per decode (one bench step): the prompt ids and the two uniform
                # tables go up; one step summary (16 + gamma_max + 8 int32)
                # comes back per step-graph replay
                "h2d_bytes_per_step": 4 * (args.prompt + 1) + 8 * 2 * 4096,
                "d2h_bytes_per_step": int(4 * (16 + args.gamma_max + 8) * results["pearl"]["replays"]
                                          / max(1, args.steps))},
        **legs,
        "gpu_launches": int(results["pearl"]["launches"]),
        "exact_cdf_fallbacks": int(results["pearl"]["fallbacks"]),
        "greedy_T0": greedy_leg,
        "roofline": rl,
        "split_pair_model": split_model,
        "run_summary": summary,
        "batch_sweep": sweep,
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def aggregate_one(r, ws):
    return aggregate({"x": r}, ws)["x"]


def summarize_legs(results, ws, sd_gammas, pearl_fixed, agg=None):
    """tokens/s of every engine leg (device time, max over ranks) and the
    speedup columns: PEARL (adaptive) over AR, over the BEST fixed-gamma SD
    (and SD at gamma 4), and over the best fixed-gamma PEARL."""
    agg = agg or {k: aggregate_one(v, ws) for k, v in results.items()}
    tps = {k: a[3] / a[0] for k, a in agg.items()}
    sd = {str(g): round(tps[f"sd{g}"], 2) for g in sd_gammas}
    sd_best_g = max(sd_gammas, key=lambda g: tps[f"sd{g}"])
    out = {
        "ar_tokens_per_s": round(tps["ar"], 2),
        "sd_by_gamma_tokens_per_s": sd,
        "sd_best_tokens_per_s": round(tps[f"sd{sd_best_g}"], 2),
        "sd_best_gamma": sd_best_g,
        "speedup_vs_ar": round(tps["pearl"] / tps["ar"], 3),
        "speedup_vs_sd": round(tps["pearl"] / tps[f"sd{sd_best_g}"], 3),
        "speedup_vs_sd_gamma4": round(tps["pearl"] / tps["sd4"], 3) if "sd4" in tps else None,
        "e2e_speedup_vs_ar": round((agg["pearl"][3] / agg["pearl"][2]) / (agg["ar"][3] / agg["ar"][2]), 3),
        "mean_accepted_tokens_per_target_fwd": round(results["pearl"]["mean_tok_per_fwd"], 3),
        "sd_mean_tokens_per_target_fwd": round(results[f"sd{sd_best_g}"]["mean_tok_per_fwd"], 3),
        "alpha_hat": None if results["pearl"]["alpha"] is None else round(results["pearl"]["alpha"], 4),
        "pearl_gamma_hist": results["pearl"].get("gamma_hist"),
        "pearl_per_decode_tokens_per_s": _spread(results["pearl"]["per_decode"]),
    }
    if pearl_fixed:
        pf = {str(g): round(tps[f"pearl{g}"], 2) for g in pearl_fixed}
        best = max(pearl_fixed, key=lambda g: tps[f"pearl{g}"])
        out.update({"pearl_fixed_by_gamma_tokens_per_s": pf, "pearl_fixed_best_gamma": best,
                    "adaptive_vs_best_fixed_pearl": round(tps["pearl"] / tps[f"pearl{best}"], 3)})
    else:
        out["pearl_tokens_per_s"] = round(tps["pearl"], 2)
    return out


def run_split(args, ws, rank, local):
    """N >= 2 (north_star placement): ranks (2i, 2i+1) form split pair i --
    the target on the even GPU, the draft on the odd one, meeting through K6
    mailboxes (NVLink peer memory, or copy-engine peer copies where the GPUs
    cannot map each other).  Each pair decodes its own prompt shard (per-pair
    prompts; per-prompt seeds as cli.py:94-96); tokens are counted once per
    pair (target ranks), time is the max over all ranks.  Target ranks also
    time single-GPU AR on the same prompts for the speedup column."""
    import datetime
    import torch
    import torch.distributed as dist
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import llama, split_pair

    gloo = dist.new_group(backend="gloo", timeout=datetime.timedelta(seconds=600))
    role, peer = split_pair.pair_roles(rank, ws)
    is_t = role == split_pair.ROLE_TARGET
    tname, dname = llama.PAIRS[args.pair]
    mc = llama.PRESETS[tname if is_t else dname]
    align = llama.AlignSpec(branch_std=args.branch_std if args.branch_std is not None else PAIR_BRANCH_STD[args.pair],
                            kappa=args.kappa)
    dev = torch.device("cuda", torch.cuda.current_device())
    shared = llama._shared_tables(mc.vocab, align, dev)
    w = llama.init_weights(mc, align, align.seed + (1 if is_t else 2), dev, shared)
    del shared
    greedy = args.temperature <= 0
    temp = 1.0 if greedy else args.temperature
    gemm = args.gemm_target if is_t else ("tcgen05" if mc.weight_bytes() > 1e9 else "cudacore")
    model = llama.LlamaModel(mc, w, gemm=gemm, max_seq=args.prompt + args.new + 2 * args.gamma_max + 16,
                             max_tokens=128 if gemm == "tcgen05" else 64, temperature=temp)
    remote = split_pair.connect_pair(model, role, peer, gamma_max=args.gamma_max, group=gloo, timeout_s=120.0)
    prompts = _prompts(args.warmup + args.steps, args.prompt, mc.vocab, seed=2000 + rank // 2)

    def cfg_for(i, g, adaptive=True):
        return pk.EngineConfig(gamma=args.gamma, max_new_tokens=args.new, seed=17 + i, greedy=g, temperature=temp,
                               adaptive_gamma=adaptive, gamma_max=args.gamma_max)

    def pearl(i, g=greedy):
        c = cfg_for(i, g)
        return pk.decode_pearl(remote, model, prompts[i], c) if is_t else pk.decode_pearl(model, remote, prompts[i], c)

    def timed(fn, clocks=False, kind="pearl"):
        for i in range(args.warmup):
            fn(i)
        torch.cuda.synchronize()
        dist.barrier(group=gloo)
        ck = Clocks(local) if clocks else None
        t0 = time.perf_counter()
        res = [fn(args.warmup + i) for i in range(args.steps)]
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = _leg_stats(res, kind, pk)
        st.update(wall_s=wall, event_s=wall)
        if not is_t:
            st["tokens"] = 0  # counted once per pair, on its target rank
        dist.barrier(group=gloo)
        return st, res, (ck.stop() if ck else None)

    try:
        pst, pres, clocks = timed(pearl, clocks=rank == 0)
        gst = timed(lambda i: pearl(i, True))[0] if args.greedy_leg and not greedy else None
    finally:
        remote.link.close()
    # single-GPU AR on the target ranks, same prompts (the speedup baseline)
    if is_t:
        ast = timed(lambda i: pk.decode_autoregressive(model, prompts[i], cfg_for(i, greedy, False)), kind="ar")[0]
    else:
        dist.barrier(group=gloo)
        dist.barrier(group=gloo)
        ast = {"tokens": 0, "device_s": 0.0, "wall_s": 0.0, "event_s": 0.0}
    rl = roofline(model, None, int(max((pst.get("gamma_hist") or {str(args.gamma): 1}).items(),
                                       key=lambda kv: kv[1])[0]), args) if is_t else None
    drl = draft_roofline(model, _peaks()[0]) if not is_t else None
    ex_bytes = {"draft_to_target_per_step": "gamma x 4 B ids + gamma x V x 4 B q-logit rows (T > 0; ids only at T=0)",
                "target_to_draft_per_step": 32}
    agg_p = aggregate({"p": pst}, ws, device="cpu", group=gloo)["p"]
    agg_a = aggregate({"a": ast}, ws, device="cpu", group=gloo)["a"]
    agg_g = aggregate({"g": gst}, ws, device="cpu", group=gloo)["g"] if gst else None
    gathered = [None] * ws
    dist.all_gather_object(gathered, {"rank": rank, "role": role, "roofline": rl, "draft_roofline": drl,
                                      "gamma_hist": pst.get("gamma_hist"), "alpha": pst["alpha"],
                                      "mean_tok": pst["mean_tok_per_fwd"], "per_decode": pst["per_decode"]},
                           group=gloo)
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return None
    pairs = ws // 2
    dp, ep, wp, tp = agg_p
    da, ea, wa, ta = agg_a
    value = tp / dp
    ar_per_pair = (ta / da) / pairs
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * wp / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts (uniform random ids), random-init weights (controlled-alignment init)",
        "config": {"workload": f"{args.pair} PEARL, {pairs} split pair(s): target GPU 2i, draft GPU 2i+1, "
                               f"batch 1 per pair, prompt {args.prompt}, {args.new} new tokens, "
                               f"{'greedy T=0' if greedy else f'T={temp:g}'}, adaptive draft length",
                   "pair": args.pair, "global_batch": pairs, "prompt_len": args.prompt, "new_tokens": args.new,
                   "parallelism": f"split pairs x{pairs} (K6 draft->target exchange per step, no collective)",
                   "gamma_max": args.gamma_max, "temperature": 0.0 if greedy else temp},
        "e2e": {"value": round(tp / wp, 2), "unit": UNIT, "h2d_bytes_per_step": 4 * (args.prompt + 1) + 8 * 4096,
                "d2h_bytes_per_step": 4 * (16 + args.gamma_max + 8)},
        "ar_tokens_per_s": round(ta / da, 2),
        "ar_tokens_per_s_per_gpu": round(ar_per_pair, 2),
        "speedup_vs_ar": round((value / pairs) / ar_per_pair, 3),
        "tokens_per_s_per_pair": round(value / pairs, 2),
        "mean_accepted_tokens_per_target_fwd": round(statistics.mean(g["mean_tok"] for g in gathered if g["role"] == "target"), 3),
        "alpha_hat": round(statistics.mean(g["alpha"] for g in gathered if g["role"] == "target"), 4),
        "pearl_gamma_hist": gathered[0]["gamma_hist"],
        "pearl_per_decode_tokens_per_s": _spread([x for g in gathered if g["role"] == "target" for x in g["per_decode"]]),
        "greedy_T0": {"tokens_per_s": round(agg_g[3] / agg_g[0], 2)} if agg_g else None,
        "exchange": ex_bytes,
        "gpu_launches": int(pst["launches"]),
        "roofline": gathered[0]["roofline"],
        "draft_roofline": gathered[1]["draft_roofline"],
        "cpu_baseline": None,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return line


def run_summaries(target, draft, timed, args):
    """the CLI's RunSummary (cli.py:65-83, 288-315) of the timed
    PEARL and SD decodes, each trace priced by the reference's step model
    (simulator.py) with t and c MEASURED on this GPU, next to the measured
    speedup -- the simulated-vs-measured comparison and the draft-run
    histogram (Fig. 2b analogue)."""
    from paper_2408_11850_b200 import metrics
    params = metrics.measured_params(target, draft)
    target.reset_adapter()
    draft.reset_adapter()
    out = {"t_draft_ms": round(params.t * 1e3, 4), "c": round(params.c, 2)}
    sd_keys = [k for k in timed if k.startswith("sd")]
    if "pearl" in timed:
        out["pearl"] = metrics.summarize_run("pearl", -1, timed["pearl"], params).to_dict()
    for k in sd_keys:
        out[k] = metrics.summarize_run("sd", int(k[2:]), timed[k], params).to_dict()
    return out


def split_pair_model(target, draft, alpha):
    """PREDICTED (not measured) tokens/s of one split pair -- draft on its own
    GPU, target on another -- from this run's own measurements:
    target window forward times t_t(M) and draft token time t_d (forward + pick)
    each timed alone on this B200, and this run's PEARL alpha-hat, through the
    stationary PEARL rate E(alpha, g) / max(t_t(g) + t_v, g t_d + t_x)
    (fastpath.pearl_tokens_per_step; t_v = K1 + commit, t_x = K6 exchange).
    Reported because this sandbox has one GPU; the split path itself is
    parity-tested (tests/test_split_gpu.py)."""
    if alpha is None:
        return None
    from paper_2408_11850_b200.fastpath import pearl_tokens_per_step
    t_t = {m: target.measure_forward_time(m) for m in (1, 4, 8, 16, 32)}
    t_d = draft.measure_forward_time(1) + 15e-6
    target.reset_adapter()
    draft.reset_adapter()
    t_v, t_x = 60e-6, 10e-6
    ks = sorted(t_t)

    def tt(m):
        for lo, hi in zip(ks, ks[1:]):
            if m <= hi:
                return t_t[lo] + (t_t[hi] - t_t[lo]) * (m - lo) / (hi - lo)
        return t_t[ks[-1]] * m / ks[-1]
    best = max(((pearl_tokens_per_step(alpha, g) / max(tt(g) + t_v, g * t_d + t_x), g)
                for g in (1, 2, 3, 4, 6, 8, 12, 16, 20, 24, 32)))
    return {"kind": "model, not a measurement (1-GPU sandbox)", "predicted_tokens_per_s": round(best[0], 1),
            "gamma": best[1], "alpha_hat": round(alpha, 4), "t_draft_ms": round(t_d * 1e3, 4),
            "t_target_ms": {str(m): round(v * 1e3, 4) for m, v in t_t.items()}}


def batch_sweep(target, draft, args, bs, greedy, temp, ws):
    """C5: B prompts decoded in lockstep (batched.py) by PEARL, SD and AR.
    PEARL and SD run at each fixed gamma of SWEEP_GAMMAS; the best of each is
    reported with its gamma (and every gamma's number).  Tokens/s of the whole
    batch from device time (the per-step host work inside it), per rank x ranks
    (ranks decode disjoint batches)."""
    import torch
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import batched
    sweep_gammas = [int(g) for g in args.sweep_gammas.split(",")] if args.sweep_gammas else list(SWEEP_GAMMAS)
    out = {}
    V = target.cfg.vocab
    for B in bs:
        prompts = _prompts(B, args.prompt, V, seed=3000 + B)
        row = {"by_gamma": {}}

        def timed(fn):
            fn()  # warm-up (graph capture)
            torch.cuda.synchronize()
            res = fn()
            toks = sum(len(r.tokens) for r in res)
            steps = [st for r in res for st in r.steps]
            return ws * toks / res[0].stats["device_s"], steps
        for kind in ("pearl", "sd"):
            best = None
            for g in sweep_gammas:
                cfg = pk.EngineConfig(gamma=g, max_new_tokens=args.new, seed=29, greedy=greedy, temperature=temp,
                                      gamma_max=max(g, args.gamma_max))
                fn = (lambda c=cfg: batched.decode_pearl_batch(draft, target, prompts, c)) if kind == "pearl" else \
                     (lambda c=cfg: batched.decode_sd_batch(draft, target, prompts, c))
                tps, steps = timed(fn)
                row["by_gamma"][f"{kind}_g{g}"] = round(tps, 2)
                if best is None or tps > best[0]:
                    best = (tps, g, pk.empirical_acceptance(steps))
            row[kind] = round(best[0], 2)
            row[kind + "_gamma"] = best[1]
            row[kind + "_alpha_hat"] = round(best[2], 4)
        cfg = pk.EngineConfig(gamma=1, max_new_tokens=args.new, seed=29, greedy=greedy, temperature=temp)
        row["ar"] = round(timed(lambda: batched.decode_autoregressive_batch(target, prompts, cfg))[0], 2)
        row["pearl_vs_ar"] = round(row["pearl"] / row["ar"], 3)
        row["pearl_vs_sd"] = round(row["pearl"] / row["sd"], 3)
        out[str(B)] = row
    return {"unit": "tokens/s (whole batch, all ranks)", "gammas_tried": list(sweep_gammas), "by_batch": out,
            "note": "lockstep engines; target/draft passes as CUDA graphs, one batched K1 launch per step; B=1 is the "
                    "single-sequence graph engine; best fixed gamma per engine"}


SWEEP_GAMMAS = (4, 8, 16)


def aggregate(results, ws, device=None, group=None):
    """(max device s, max event s, max wall s, sum tokens) per engine over ranks."""
    import torch
    import torch.distributed as dist
    if device is None:
        device = "cpu" if ws > 1 and dist.get_backend() == "gloo" else "cuda"
    agg = {}
    for kind, r in results.items():
        vals = torch.tensor([r["device_s"], r["event_s"], r["wall_s"], float(r["tokens"])], device=device,
                            dtype=torch.float64)
        if ws > 1:
            mx = vals.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
            sm = vals.clone()
            dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=group)
            agg[kind] = (mx[0].item(), mx[1].item(), mx[2].item(), sm[3].item())
        else:
            agg[kind] = tuple(vals.tolist())
    return agg


def _forward_time(model, M, ctx, n=10):
    """CUDA-event time of one M-token window forward at position ctx, the
    forward captured as a CUDA graph and replayed back to back (as inside a
    decode step graph)."""
    import torch
    toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
    pos = torch.tensor([ctx], dtype=torch.int32, device="cuda")
    out = torch.empty(M, model.cfg.vocab, dtype=torch.float32, device="cuda")
    for _ in range(2):
        model.forward(toks, M, pos, 0, out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        model.forward(toks, M, pos, 0, out)
    for _ in range(2):
        g.replay()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        g.replay()
    e.record()
    e.synchronize()
    model.reset_adapter()
    return s.elapsed_time(e) / 1e3 / n


def _forward_bytes(c, M, ctx):
    return c.weight_bytes() + c.kv_bytes_per_token() * (ctx + M) + 4 * M * c.vocab


def window_frac(target, M, args):
    ctx = args.prompt + args.new // 2
    t = _forward_time(target, M, ctx)
    return {"ms": round(t * 1e3, 4), "frac": round(_forward_bytes(target.cfg, M, ctx) / t / 1e9 / _peaks()[0], 4)}


def roofline(target, draft, gamma, args):
    """Dominant kernel sequence = one target window forward (M = gamma tokens).

    Algorithmic bytes per forward = bf16 weights + KV read over the context +
    fp32 logits written; time = CUDA-event average of the forward (graph
    replays on its stream), after warm-up.
    """
    peak, src = _peaks()
    M = max(1, int(gamma))
    ctx = args.prompt + args.new // 2
    t = _forward_time(target, M, ctx)
    c = target.cfg
    byts = _forward_bytes(c, M, ctx)
    achieved = byts / t / 1e9
    # ncu DRAM bytes of one forward (profiles/traffic.json) at this window, else
    # at the nearest captured window of this model (weights dominate: 7B M=16
    # 13.53 GB, M=20 13.56 GB), named in traffic_window
    tab = {k: v for k, v in _traffic().items() if k.startswith(f"{c.name}_M")}
    tr, tr_m = None, None
    if tab:
        key = min(tab, key=lambda k: abs(int(k.rsplit("_M", 1)[1]) - M))
        tr, tr_m = tab[key], int(key.rsplit("_M", 1)[1])
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": tr, "traffic_window": tr_m,
            "kernel": f"target window forward ({c.name}, M={M}, ctx={ctx}, {args.gemm_target} GEMMs)",
            "bytes_per_launch": int(byts), "ms_per_launch": round(t * 1e3, 4), "peak_source": src,
            "gemm_kernel": gemm_roofline(target, M, peak) if args.gemm_target == "tcgen05" else None,
            "draft_forward": draft_roofline(draft, peak) if draft is not None else None}


def draft_roofline(draft, peak):
    """K2 chain: one draft token forward (M=1, logits for the pick) as a CUDA
    graph replayed back to back, CUDA-event timed; bytes = bf16 weights + KV."""
    import torch
    toks = torch.full((1,), 5, dtype=torch.int32, device="cuda")
    pos = torch.tensor([192], dtype=torch.int32, device="cuda")
    out = torch.empty(1, draft.cfg.vocab, device="cuda")
    for _ in range(3):
        draft.forward(toks, 1, pos, 2, out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        draft.forward(toks, 1, pos, 2, out)
    n = 50
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        g.replay()
    e.record()
    e.synchronize()
    t = s.elapsed_time(e) / 1e3 / n
    c = draft.cfg
    byts = c.weight_bytes() + c.kv_bytes_per_token() * 193 + 4 * c.vocab
    draft.reset_adapter()
    return {"kernel": f"draft token forward ({c.name}, {draft.gemm}, CUDA graph)", "bytes_per_launch": int(byts),
            "us_per_launch": round(t * 1e6, 2), "achieved": round(byts / t / 1e9, 1),
            "frac": round(byts / t / 1e9 / peak, 4)}


def gemm_roofline(target, M, peak):
    """K3 alone (tc_gemm_kernel, ~80-90% of a forward in the ncu launch lists):
    layer 0's four weight matrices of the target (qkv, o, gate_up, down) at M
    tokens, launched back to back on one stream, CUDA-event timed; achieved =
    weight bytes streamed / time."""
    import torch
    from paper_2408_11850_b200 import _lib
    lib = _lib.load()
    L = target.w["layers"][0]
    mats = [L["wqkv"], L["wo"], L["w_gate_up"], L["w_down"]]
    xs = [torch.randn(M, w.shape[1], device="cuda").to(torch.bfloat16) for w in mats]
    ys = [torch.empty(M, w.shape[0], device="cuda") for w in mats]
    st = torch.cuda.current_stream().cuda_stream

    def once():
        for w, x, y in zip(mats, xs, ys):
            _lib.check(lib.pearl_gemm(1, w.data_ptr(), x.data_ptr(), y.data_ptr(), M, w.shape[0], w.shape[1], 0, st),
                       "pearl_gemm")
    for _ in range(3):
        once()
    n = 20
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        once()
    e.record()
    e.synchronize()
    t = s.elapsed_time(e) / 1e3 / (4 * n)
    byts = sum(w.numel() * 2 for w in mats) / 4
    return {"kernel": "tc_gemm_kernel (layer-0 qkv / o / gate_up / down, back to back)", "M": M,
            "bytes_per_launch": int(byts), "us_per_launch": round(t * 1e6, 2),
            "achieved": round(byts / t / 1e9, 1), "frac": round(byts / t / 1e9 / peak, 4)}


def cpu_baseline(target, draft, prompt, args, greedy, temp):
    """The reference algorithm's CPU path on the host cores, bounded sample."""
    import torch
    from oracle import engine as oe
    from oracle.llama import OracleLlama
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    n_new = args.cpu_new
    P = min(len(prompt), args.cpu_prompt)
    mt = OracleLlama(target.cfg, _to_cpu(target.w), device="cpu", bf16_points=True, max_seq=P + n_new + 64,
                     mm_dtype=torch.bfloat16, temperature=temp)
    md = OracleLlama(draft.cfg, _to_cpu(draft.w), device="cpu", bf16_points=True, max_seq=P + n_new + 64,
                     mm_dtype=torch.bfloat16, temperature=temp)
    t0 = time.perf_counter()
    toks, steps = oe.decode_pearl(md, mt, prompt[:P], args.gamma, n_new, seed=17, greedy=greedy)
    dt = time.perf_counter() - t0
    del mt, md
    return {"value": round(len(toks) / dt, 4), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"oracle decode_pearl (pearl_lab engines.py restated) + PyTorch CPU bf16 Llama, "
                      f"{target.cfg.name}/{draft.cfg.name}, prompt {P}, {len(toks)} new tokens, gamma {args.gamma}",
            "seconds": round(dt, 2)}


def _to_cpu(w):
    out = {k: v.cpu() for k, v in w.items() if k != "layers"}
    out["layers"] = [{k: v.cpu() for k, v in L.items()} for L in w["layers"]]
    return out


def run_reference(args):
    """--impl reference: the CPU port alone (rank 0 only)."""
    ws, rank, local = _dist()
    if rank != 0:
        return None
    import torch
    from oracle import engine as oe
    from oracle.llama import OracleLlama
    from paper_2408_11850_b200.llama import AlignSpec, PRESETS, PAIRS, init_weights, _shared_tables
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    tname, dname = PAIRS[args.pair]
    tc, dc = PRESETS[tname], PRESETS[dname]
    align = AlignSpec(branch_std=args.branch_std if args.branch_std is not None else PAIR_BRANCH_STD[args.pair],
                      kappa=args.kappa)
    # weights are generated where it is fast (the GPU when present: same
    # values as the GPU arm) and then moved to host memory; only the CPU
    # decode below is timed.
    gen_dev = "cuda" if torch.cuda.is_available() else "cpu"
    shared = _shared_tables(tc.vocab, align, gen_dev)
    tw = _to_cpu(init_weights(tc, align, align.seed + 1, gen_dev, shared))
    dw = _to_cpu(init_weights(dc, align, align.seed + 2, gen_dev, shared))
    del shared
    greedy = args.temperature <= 0
    temp = 1.0 if greedy else args.temperature
    # the GPU arm's workload (prompt, new tokens, pair, temperature), one
    # decode per step; the reference engine drafts a fixed gamma (it has no
    # planner): the GPU arm's best fixed gamma on this pair
    P, N, g = args.prompt, args.new, args.ref_gamma
    mt = OracleLlama(tc, tw, device="cpu", max_seq=P + N + 2 * g + 64, mm_dtype=torch.bfloat16, temperature=temp)
    md = OracleLlama(dc, dw, device="cpu", max_seq=P + N + 2 * g + 64, mm_dtype=torch.bfloat16, temperature=temp)
    prompts = _prompts(args.warmup + args.steps, P, tc.vocab, seed=1000)
    for i in range(min(args.warmup, 1)):
        oe.decode_pearl(md, mt, prompts[i], g, 2, seed=i, greedy=greedy)
    t0 = time.perf_counter()
    toks = 0
    for i in range(args.steps):
        out, _ = oe.decode_pearl(md, mt, prompts[args.warmup + i], g, N, seed=17 + i, greedy=greedy)
        toks += len(out)
    dt = time.perf_counter() - t0
    v = toks / dt
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic prompts, random-init weights",
            "config": {"workload": f"{args.pair} PEARL (reference engine restated, fixed gamma {g}) on host CPU "
                                   f"cores, batch 1, prompt {P}, {N} new tokens, "
                                   f"{'greedy T=0' if greedy else f'T={temp:g}'}",
                       "pair": args.pair, "global_batch": 1, "prompt_len": P, "new_tokens": N, "gamma": g,
                       "temperature": 0.0 if greedy else temp},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} x decode_pearl of {N} tokens, prompt {P}, gamma {g} "
                                       f"(oracle/engine.py + PyTorch CPU bf16 Llama)"},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # 20 prompts (the driver's sample): PEARL's per-decode spread is wide (5 prompts
    # gave 1388-1681 tok/s for one code / calibration pair; 20 give 1311-1332)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pair", default="llama2-7b/68m")
    ap.add_argument("--gamma", type=int, default=4, help="initial draft length of adaptive PEARL")
    ap.add_argument("--sd-gammas", default="4,8,16,20,24,32", help="fixed draft lengths of the vanilla SD legs (the best of them is the SD baseline)")
    ap.add_argument("--pearl-gammas", default="4,8,16,24", help="fixed draft lengths of the fixed-gamma PEARL legs")
    ap.add_argument("--gamma-max", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--new", type=int, default=128)
    ap.add_argument("--temperature", type=float, default=1.0)
    ap.add_argument("--greedy-leg", type=int, default=1, help="also time T=0 (BASELINE configs[1] asks T in {0, 1})")
    ap.add_argument("--live-calibration", action="store_true",
                    help="measure the adaptive planner's step-time table now instead of loading profiles/")
    ap.add_argument("--branch-std", type=float, default=None,
                    help="alignment knob (default per pair, calibrated to alpha-hat ~0.9 at T=1: tools/calib_alpha.py)")
    ap.add_argument("--kappa", type=float, default=13.0)
    ap.add_argument("--gemm-target", default="tcgen05")
    ap.add_argument("--draft-sms", type=int, default=None,
                    help="green-context SMs for PEARL's concurrent draft (default per pair, PAIR_DRAFT_SMS)")
    ap.add_argument("--cpu-new", type=int, default=16, help="new tokens of the in-bench cpu_baseline sample")
    ap.add_argument("--ref-gamma", type=int, default=16,
                    help="--impl reference: the CPU reference engine's fixed draft length")
    ap.add_argument("--cpu-prompt", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>=2: co-resident replicas per GPU instead of split pairs")
    ap.add_argument("--sweep-gammas", default=",".join(str(g) for g in SWEEP_GAMMAS),
                    help="C5: fixed draft lengths tried per engine and batch size")
    ap.add_argument("--batch-sweep", default="1,4,16,32",
                    help="C5: comma-separated batch sizes decoded in lockstep (empty string: skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
