"""Where a batched step's time goes: slot-mode forwards vs single-sequence ones, and the host loop.

    python tools/batch_prof.py [B]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_11850_b200 as pk
from paper_2408_11850_b200 import llama, batched
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
target, draft = llama.build_pair("llama2-7b/68m", gemm_target="tcgen05", align=llama.AlignSpec(branch_std=5e-4),
                                 max_seq=400, max_tokens=128, n_slots=B)
dev = target.device
def timed(fn, n=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
for M in (1, B):
    toks = torch.full((M,), 5, dtype=torch.int32, device=dev)
    slots = torch.arange(M, dtype=torch.int32, device=dev) % B
    pos = torch.full((M,), 192, dtype=torch.int32, device=dev)
    out = torch.empty(M, target.cfg.vocab, device=dev)
    p1 = torch.tensor([192], dtype=torch.int32, device=dev)
    print(f"M={M}: single-seq forward {timed(lambda: target.forward(toks, M, p1, 0, out)):.3f} ms | "
          f"slot forward (M seqs x 1 token) {timed(lambda: target.forward_slots(toks, M, slots, pos, out)):.3f} ms | "
          f"draft slot forward {timed(lambda: draft.forward_slots(toks, M, slots, pos, out)):.3f} ms", flush=True)
prompts = [np.random.default_rng(i).integers(2, 32000, 128).tolist() for i in range(B)]
for kind in ("ar", "sd", "pearl"):
    cfg = pk.EngineConfig(gamma=4, max_new_tokens=64, seed=1, greedy=False)
    fn = {"ar": lambda: batched.decode_autoregressive_batch(target, prompts, cfg),
          "sd": lambda: batched.decode_sd_batch(draft, target, prompts, cfg),
          "pearl": lambda: batched.decode_pearl_batch(draft, target, prompts, cfg)}[kind]
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fn()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st = res[0].stats
    toks = sum(len(r.tokens) for r in res)
    print(f"{kind} B={B}: {st['steps']} steps, device_s {st['device_s']*1e3:.1f} ms (prefill {st['prefill_s']*1e3:.1f}), "
          f"wall {wall*1e3:.1f} ms, {toks / st['device_s']:.0f} tok/s; per step {(st['device_s']-st['prefill_s'])/st['steps']*1e3:.2f} ms",
          flush=True)
