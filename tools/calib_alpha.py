"""Measured acceptance rate alpha-hat of a random-init pair vs the alignment
knob branch_std (T=1, SD gamma=4, 2 prompts x 64 new tokens)."""
import sys, os, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_11850_b200 as pk
from paper_2408_11850_b200 import llama
pair = sys.argv[1]
stds = [float(s) for s in sys.argv[2].split(",")]
prompt = int(sys.argv[3]) if len(sys.argv) > 3 else 128
for sd in stds:
    t, d = llama.build_pair(pair, gemm_target="tcgen05", align=llama.AlignSpec(branch_std=sd), max_seq=prompt + 64 + 40)
    rng = np.random.default_rng(5)
    steps = []
    for i in range(2):
        p = rng.integers(2, t.cfg.vocab, prompt).tolist()
        r = pk.decode_sd(d, t, p, pk.EngineConfig(gamma=4, max_new_tokens=64, seed=i))
        steps += list(r.steps)
    print(f"{pair} branch_std={sd:g}: alpha_hat={pk.empirical_acceptance(steps):.3f}", flush=True)
    t.close(); d.close(); del t, d; gc.collect(); torch.cuda.empty_cache()
