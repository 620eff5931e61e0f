"""Benchmark: PEARL decoding on B200 (BASELINE.json metric, configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (configs[1] of BASELINE.json): Llama-2-7B target + Llama-68M draft,
random-init bf16 weights (controlled-alignment init, llama.py), batch 1,
synthetic 128-token prompts, 128 new tokens, draft and target co-resident on
one B200 (N=1).  A *step* is one ``decode_pearl`` call (prefill + decode of
128 tokens) through the public API.  AR and fixed-gamma SD run on the same
kernels in the same process for the speedup columns.

Metric: generated tokens/s (whole job, all ranks), plus speedup vs AR and
vs vanilla SD and mean accepted tokens per target forward.
  value = tokens / device time of the decode graphs (inputs resident)
  e2e   = tokens / wall time of the public API calls (host prompt in, host
          tokens out: H2D of prompt + uniform tables, D2H of step summaries)
Weights (13.6 GB) exceed L2 (126 MB), so every forward streams from HBM.

N>1: one process per GPU (torchrun); each rank runs its own co-resident
draft/target replica on its own prompt shard (replicas only, no data-path
collective); value = all ranks' tokens / max-over-ranks time.

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


def run_gpu(args):
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
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import _lib, llama

    align = llama.AlignSpec(branch_std=args.branch_std if args.branch_std is not None else PAIR_BRANCH_STD[args.pair],
                            kappa=args.kappa)
    sweep_bs = [int(b) for b in args.batch_sweep.split(",") if b] if args.batch_sweep else []
    target, draft = llama.build_pair(args.pair, gemm_target=args.gemm_target, align=align,
                                     n_slots=max([1] + sweep_bs),
                                     max_seq=args.prompt + args.new + 2 * args.gamma_max + 16, max_tokens=128,
                                     temperature=1.0 if args.temperature <= 0 else args.temperature,
                                     draft_sms=args.draft_sms if args.draft_sms is not None
                                     else int(os.environ.get("PEARL_DRAFT_SMS", PAIR_DRAFT_SMS[args.pair])))
    greedy = args.temperature <= 0
    temp = 1.0 if greedy else args.temperature
    V = target.cfg.vocab
    draft_sms_used = getattr(target, "green_partition", (None, None, 0, 0))[2]
    prompts = _prompts(args.warmup + args.steps, args.prompt, V, seed=1000 + rank)

    def cfg_for(gamma, seed, adaptive=False):
        return pk.EngineConfig(gamma=gamma, max_new_tokens=args.new, seed=seed, greedy=greedy, temperature=temp,
                               adaptive_gamma=adaptive, gamma_max=args.gamma_max)

    pearl_gamma = args.gamma

    def run(kind, i):
        if kind == "pearl":
            return pk.decode_pearl(draft, target, prompts[i], cfg_for(pearl_gamma, 17 + i, not args.fixed_gamma))
        if kind == "sd":
            return pk.decode_sd(draft, target, prompts[i], cfg_for(args.sd_gamma, 17 + i))
        if kind in ("sd8", "sd16"):
            return pk.decode_sd(draft, target, prompts[i], cfg_for(int(kind[2:]), 17 + i))
        return pk.decode_autoregressive(target, prompts[i], cfg_for(1, 17 + i))

    results = {}
    timed_results = {}
    clocks = None
    for kind in ("ar", "sd", "sd8", "sd16", "pearl"):  # PEARL last: its clocks are sampled
        for i in range(args.warmup):
            run(kind, i)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        if kind == "pearl":
            clocks = Clocks(local)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        res = [run(kind, args.warmup + i) for i in range(args.steps)]
        ev1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ev_s = ev0.elapsed_time(ev1) / 1e3
        if kind == "pearl":
            clocks = clocks.stop()
        toks = sum(len(r.tokens) for r in res)
        dev = sum(r.stats["device_s"] for r in res)
        timed_results[kind] = res
        steps = [s for r in res for s in r.steps]
        results[kind] = dict(tokens=toks, device_s=dev, wall_s=wall, event_s=ev_s,
                             launches=sum(r.stats["launches"] for r in res),
                             replays=sum(r.stats.get("replays", 0) for r in res),
                             mean_tok_per_fwd=pk.mean_tokens_per_target_forward(steps),
                             alpha=pk.empirical_acceptance(steps) if kind != "ar" else None,
                             gamma=res[0].stats.get("gamma"),
                             gammas=sorted(set(g for r in res for g in r.stats.get("gammas", []))),
                             fallbacks=sum(r.stats.get("fallbacks", 0) for r in res))
    # max over ranks of the timed region, sum of tokens
    agg = aggregate(results, ws)
    # roofline of the dominant kernel sequence: one target window forward
    rl = roofline(target, draft, args.gamma, args)
    summary = run_summaries(target, draft, timed_results, args)
    split_model = split_pair_model(target, draft, results["pearl"]["alpha"]) if ws == 1 else None
    target_bytes, draft_bytes = target.cfg.weight_bytes(), draft.cfg.weight_bytes()
    sweep = batch_sweep(target, draft, args, sweep_bs, greedy, temp, ws) if sweep_bs else None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(target, draft, prompts[0], args, greedy, temp)
    split = None
    if ws >= 2 and ws % 2 == 0 and not args.no_split:
        # the co-resident replicas are freed first: a split rank hosts one model
        del target, draft
        split = split_leg(args, ws, rank, greedy, temp, agg["ar"])
    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return None
    wbytes = target_bytes + draft_bytes
    dp, ep, wp, tp = agg["pearl"]
    da, ea, wa, ta = agg["ar"]
    ds_, es, wsd, ts_ = agg["sd"]
    value = tp / dp
    line = {
        "metric": METRIC,
        "value": round(value, 2),
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
            "workload": f"{args.pair} PEARL, batch 1, prompt {args.prompt}, {args.new} new tokens, "
                        f"{'greedy T=0' if greedy else f'T={temp}'}, draft+target co-resident per GPU",
            "pair": args.pair, "global_batch": ws, "prompt_len": args.prompt, "new_tokens": args.new,
            "gamma": results["pearl"]["gammas"] if not args.fixed_gamma else args.gamma,
            "adaptive_gamma": not args.fixed_gamma,
            "sd_gamma": args.sd_gamma, "temperature": 0.0 if greedy else temp,
            "target_gemm": args.gemm_target, "parallelism": f"replicas x{ws}",
            "draft_sms": draft_sms_used,
            "l2": f"weights {wbytes / 1e9:.2f} GB vs 126 MB L2: "
                  + ("every forward streams HBM (no flush needed)" if wbytes > 126e6 else "L2-resident (tiny pair)"),
        },
        "e2e": {"value": round(tp / ep, 2), "unit": UNIT,
                # per decode (one bench step): the prompt ids and the two uniform
                # tables go up; one step summary (16 + gamma_max + 8 int32)
                # comes back per step-graph replay
                "h2d_bytes_per_step": 4 * (args.prompt + 1) + 8 * 2 * 4096,
                "d2h_bytes_per_step": int(4 * (16 + args.gamma_max + 8) * results["pearl"]["replays"]
                                          / max(1, args.steps))},
        "ar_tokens_per_s": round(ta / da, 2),
        "sd_tokens_per_s": round(ts_ / ds_, 2),
        "speedup_vs_ar": round((tp / dp) / (ta / da), 3),
        "speedup_vs_sd": round((tp / dp) / (ts_ / ds_), 3),
        "sd_best_tokens_per_s": round(max(agg[k][3] / agg[k][0] for k in ("sd", "sd8", "sd16")), 2),
        "sd_by_gamma_tokens_per_s": {str(args.sd_gamma): round(ts_ / ds_, 2),
                                     "8": round(agg["sd8"][3] / agg["sd8"][0], 2),
                                     "16": round(agg["sd16"][3] / agg["sd16"][0], 2)},
        "e2e_speedup_vs_ar": round((tp / ep) / (ta / ea), 3),
        "mean_accepted_tokens_per_target_fwd": round(results["pearl"]["mean_tok_per_fwd"], 3),
        "sd_mean_tokens_per_target_fwd": round(results["sd"]["mean_tok_per_fwd"], 3),
        "alpha_hat": None if results["pearl"]["alpha"] is None else round(results["pearl"]["alpha"], 4),
        "sd_alpha_hat": None if results["sd"]["alpha"] is None else round(results["sd"]["alpha"], 4),
        "gpu_launches": int(results["pearl"]["launches"]),
        "exact_cdf_fallbacks": int(results["pearl"]["fallbacks"]),
        "roofline": rl,
        "split_pair": split,
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
    for kind in ("pearl", "sd"):
        if kind in timed:
            out[kind] = metrics.summarize_run(kind, args.gamma if kind == "sd" else -1, timed[kind], params).to_dict()
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


def split_leg(args, ws, rank, greedy, temp, ar_agg):
    """N >= 2: ranks (2i, 2i+1) form split pair i -- the target on the even
    GPU, the draft on the odd one, meeting through K6 mailboxes (NVLink peer
    memory).  Each pair decodes its own prompts; tokens are counted once per
    pair (target ranks), time is the max over all ranks.

    Guarded: every rank-local failure (including a K6 wait timing out) is
    caught, all ranks agree on success through one collective, and the leg
    reports {"error": ...} instead of taking the replica line down with it."""
    import datetime
    import torch
    import torch.distributed as dist
    import paper_2408_11850_b200 as pk
    gloo = dist.new_group(backend="gloo", timeout=datetime.timedelta(seconds=240))
    err, local = None, None
    try:
        local = _split_local(args, ws, rank, greedy, temp, gloo)
    except Exception as ex:  # noqa: BLE001 -- reported, never fatal
        err = f"rank {rank}: {type(ex).__name__}: {str(ex)[:200]}"
    flag = torch.tensor([1.0 if err else 0.0])
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=gloo)
    if flag.item() > 0:
        return {"error": err or "a peer rank failed"}
    one, steps, gammas = local
    d, e, wl, t = aggregate(one, ws)["pearl"]
    ar_tps_per_gpu = ar_agg[3] / ar_agg[0] / ws
    return {"pairs": ws // 2, "placement": "target on even GPU, draft on odd GPU, K6 NVLink mailboxes",
            "tokens_per_s": round(t / d, 2), "e2e_tokens_per_s": round(t / e, 2),
            "tokens_per_s_per_pair": round(t / d / (ws // 2), 2),
            "speedup_vs_single_gpu_ar": round(t / d / (ws // 2) / ar_tps_per_gpu, 3),
            "mean_accepted_tokens_per_target_fwd": round(pk.mean_tokens_per_target_forward(steps), 3),
            "alpha_hat": round(pk.empirical_acceptance(steps), 4), "gammas": gammas}


def _split_local(args, ws, rank, greedy, temp, gloo):
    import gc
    import torch
    import torch.distributed as dist
    import paper_2408_11850_b200 as pk
    from paper_2408_11850_b200 import llama, split_pair

    gc.collect()
    torch.cuda.empty_cache()
    role, peer = split_pair.pair_roles(rank, ws)
    tname, dname = llama.PAIRS[args.pair]
    mc = llama.PRESETS[tname if role == split_pair.ROLE_TARGET else dname]
    need = mc.weight_bytes() * 1.1 + (2 << 30)
    ok = torch.tensor([1.0 if torch.cuda.mem_get_info()[0] > need else 0.0])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=gloo)
    if ok.item() < 1:
        raise RuntimeError("not enough free device memory after the replica leg")
    align = llama.AlignSpec(branch_std=args.branch_std if args.branch_std is not None else PAIR_BRANCH_STD[args.pair],
                            kappa=args.kappa)
    dev = torch.device("cuda", torch.cuda.current_device())
    shared = llama._shared_tables(mc.vocab, align, dev)
    is_t = role == split_pair.ROLE_TARGET
    w = llama.init_weights(mc, align, align.seed + (1 if is_t else 2), dev, shared)
    del shared
    gemm = args.gemm_target if is_t else ("tcgen05" if mc.weight_bytes() > 1e9 else "cudacore")
    model = llama.LlamaModel(mc, w, gemm=gemm, max_seq=args.prompt + args.new + 2 * args.gamma_max + 16,
                             max_tokens=64, temperature=1.0 if greedy else temp)
    remote = split_pair.connect_pair(model, role, peer, gamma_max=args.gamma_max, group=gloo, timeout_s=60.0)
    prompts = _prompts(args.warmup + args.steps, args.prompt, mc.vocab, seed=2000 + rank // 2)

    def run(i):
        cfg = pk.EngineConfig(gamma=args.gamma, max_new_tokens=args.new, seed=17 + i, greedy=greedy, temperature=temp,
                              adaptive_gamma=not args.fixed_gamma, gamma_max=args.gamma_max)
        return pk.decode_pearl(remote, model, prompts[i], cfg) if is_t else pk.decode_pearl(model, remote, prompts[i],
                                                                                             cfg)

    try:
        for i in range(args.warmup):
            run(i)
        torch.cuda.synchronize()
        dist.barrier(group=gloo)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        res = [run(args.warmup + i) for i in range(args.steps)]
        ev1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    finally:
        remote.link.close()
    toks = sum(len(r.tokens) for r in res) if is_t else 0
    steps = [s for r in res for s in r.steps]
    one = {"pearl": dict(device_s=sum(r.stats["device_s"] for r in res), event_s=ev0.elapsed_time(ev1) / 1e3,
                         wall_s=wall, tokens=toks)}
    return one, steps, sorted(set(g for r in res for g in r.stats.get("gammas", [])))


def aggregate(results, ws, device=None):
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
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = vals.clone()
            dist.all_reduce(sm, op=dist.ReduceOp.SUM)
            agg[kind] = (mx[0].item(), mx[1].item(), mx[2].item(), sm[3].item())
        else:
            agg[kind] = tuple(vals.tolist())
    return agg


def roofline(target, draft, gamma, args):
    """Dominant kernel sequence = one target window forward (M = gamma tokens).

    Algorithmic bytes per forward = bf16 weights + KV read over the context +
    fp32 logits written; time = CUDA-event average of the forward on its
    stream, after warm-up.
    """
    import torch
    peak, src = _peaks()
    M = max(1, int(gamma))
    ctx = args.prompt + args.new // 2
    toks = torch.full((M,), 5, dtype=torch.int32, device="cuda")
    pos = torch.tensor([ctx], dtype=torch.int32, device="cuda")
    out = torch.empty(M, target.cfg.vocab, dtype=torch.float32, device="cuda")
    for _ in range(3):
        target.forward(toks, M, pos, 0, out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    s.record()
    for _ in range(n):
        target.forward(toks, M, pos, 0, out)
    e.record()
    e.synchronize()
    t = s.elapsed_time(e) / 1e3 / n
    c = target.cfg
    byts = c.weight_bytes() + c.kv_bytes_per_token() * (ctx + M) + 4 * M * c.vocab
    achieved = byts / t / 1e9
    tr = _traffic().get(f"{c.name}_M{M}")
    target.reset_adapter()
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": tr,
            "kernel": f"target window forward ({c.name}, M={M}, ctx={ctx}, {args.gemm_target} GEMMs)",
            "bytes_per_launch": int(byts), "ms_per_launch": round(t * 1e3, 4), "peak_source": src,
            "gemm_kernel": gemm_roofline(target, M, peak) if args.gemm_target == "tcgen05" else None,
            "draft_forward": draft_roofline(draft, peak)}


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
    P = args.cpu_prompt
    mt = OracleLlama(tc, tw, device="cpu", max_seq=P + args.cpu_new + 64, mm_dtype=torch.bfloat16, temperature=temp)
    md = OracleLlama(dc, dw, device="cpu", max_seq=P + args.cpu_new + 64, mm_dtype=torch.bfloat16, temperature=temp)
    prompts = _prompts(args.warmup + args.steps, P, tc.vocab, seed=1000)
    for i in range(min(args.warmup, 1)):
        oe.decode_pearl(md, mt, prompts[i], args.gamma, 2, seed=i, greedy=greedy)
    t0 = time.perf_counter()
    toks = 0
    for i in range(args.steps):
        out, _ = oe.decode_pearl(md, mt, prompts[args.warmup + i], args.gamma, args.cpu_new, seed=17 + i,
                                 greedy=greedy)
        toks += len(out)
    dt = time.perf_counter() - t0
    v = toks / dt
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * dt / args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic prompts, random-init weights",
            "config": {"workload": f"{args.pair} PEARL on host CPU cores, bounded sample", "pair": args.pair,
                       "prompt_len": P, "new_tokens": args.cpu_new, "gamma": args.gamma},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} x decode_pearl of {args.cpu_new} tokens, prompt {P}"},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pair", default="llama2-7b/68m")
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--sd-gamma", type=int, default=4)
    ap.add_argument("--gamma-max", type=int, default=32)
    ap.add_argument("--fixed-gamma", action="store_true", help="PEARL with fixed --gamma instead of adaptive")
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--new", type=int, default=128)
    ap.add_argument("--temperature", type=float, default=1.0)
    ap.add_argument("--branch-std", type=float, default=None,
                    help="alignment knob (default per pair, calibrated to alpha-hat ~0.9 at T=1: tools/calib_alpha.py)")
    ap.add_argument("--kappa", type=float, default=13.0)
    ap.add_argument("--gemm-target", default="tcgen05")
    ap.add_argument("--draft-sms", type=int, default=None,
                    help="green-context SMs for PEARL's concurrent draft (default per pair, PAIR_DRAFT_SMS)")
    ap.add_argument("--cpu-new", type=int, default=16)
    ap.add_argument("--cpu-prompt", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-split", action="store_true", help="N>=2: skip the split-pair (draft GPU / target GPU) leg")
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
