"""Host-side profile of decode_pearl / decode_sd (graph captures, table refills, planner)."""
import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_11850_b200 as pk
from paper_2408_11850_b200 import llama, fastpath
pair = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b/68m"
align = llama.AlignSpec(branch_std=5e-4)
target, draft = llama.build_pair(pair, gemm_target="tcgen05", align=align, max_seq=128 + 128 + 64 + 16, max_tokens=64)
V = target.cfg.vocab
rng = np.random.default_rng(1000)
prompts = [rng.integers(2, V, 128).tolist() for _ in range(12)]
cfg = lambda i: pk.EngineConfig(gamma=4, max_new_tokens=128, seed=17 + i, adaptive_gamma=True, gamma_max=24)
def ngraphs():
    return sum(len(rt.graphs) for rt in target.__dict__.get("_pearl_runtimes", {}).values())
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = pk.decode_pearl(draft, target, prompts[i], cfg(i))
    torch.cuda.synchronize(); w = time.perf_counter() - t0
    print(f"decode {i}: wall {w*1e3:.1f} ms device {r.stats['device_s']*1e3:.1f} ms steps {len(r.steps)} graphs {ngraphs()} "
          f"gammas {sorted(set(r.stats['gammas']))}", flush=True)
for rt in target.__dict__.get("_pearl_runtimes", {}).values():
    print("graph keys:", sorted(k[:4] for k in rt.graphs))
pr = cProfile.Profile()
pr.enable()
for i in range(8, 10):
    pk.decode_pearl(draft, target, prompts[i], cfg(i))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
