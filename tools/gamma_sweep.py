"""PEARL vs SD vs AR over draft lengths on one pair (1 GPU, co-resident)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_11850_b200 as pk
from paper_2408_11850_b200 import llama

pair = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b/68m"
T = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
bs = float(sys.argv[3]) if len(sys.argv) > 3 else 5e-4
target, draft = llama.build_pair(pair, gemm_target="tcgen05", align=llama.AlignSpec(branch_std=bs), max_seq=512,
                                 max_tokens=64)
V = target.cfg.vocab
rng = np.random.default_rng(0)
prompts = [rng.integers(2, V, 128).tolist() for _ in range(4)]
greedy = T <= 0
def run(kind, gamma, adaptive=False):
    toks = 0; dev = 0.0; steps = []
    for i, p in enumerate(prompts):
        cfg = pk.EngineConfig(gamma=gamma, max_new_tokens=128, seed=i, greedy=greedy, temperature=1.0 if greedy else T,
                              adaptive_gamma=adaptive, gamma_max=32)
        f = {"pearl": lambda: pk.decode_pearl(draft, target, p, cfg), "sd": lambda: pk.decode_sd(draft, target, p, cfg),
             "ar": lambda: pk.decode_autoregressive(target, p, cfg)}[kind]
        f()  # warm (graph capture)
        r = f()
        toks += len(r.tokens); dev += r.stats["device_s"]; steps += list(r.steps)
    return dict(kind=kind, gamma=gamma if not adaptive else f"adaptive({r.stats.get('gamma')})", tok_s=round(toks / dev, 1),
                tok_per_step=round(pk.mean_tokens_per_target_forward(steps), 3),
                alpha=None if kind == "ar" else round(pk.empirical_acceptance(steps), 3))
print(json.dumps(run("ar", 1)), flush=True)
for g in (4, 8, 16, 32):
    print(json.dumps(run("sd", g)), flush=True)
    print(json.dumps(run("pearl", g)), flush=True)
print(json.dumps(run("pearl", 4, adaptive=True)), flush=True)
print("t_target(M=1)", target.measure_forward_time(1), "t_draft", draft.measure_forward_time(1))
