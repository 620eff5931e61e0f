"""Per-step device times: draft block alone, target window alone, and the
PEARL / SD step graphs (concurrency and contention between the two models)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_11850_b200 import llama, fastpath, _lib, _device
pair = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b/68m"
gammas = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4, 8, 12, 16, 24]
dg = os.environ.get("DRAFT_GEMM", "cudacore")
target, draft = llama.build_pair(pair, gemm_target="tcgen05", gemm_draft=dg, align=llama.AlignSpec(branch_std=5e-4),
                                 max_seq=600, max_tokens=64)
print(f"{pair}: draft gemm {dg}: draft fwd {draft.measure_forward_time(1)*1e3:.3f} ms, target fwd M=1 "
      f"{target.measure_forward_time(1)*1e3:.3f} ms", flush=True)
rt = fastpath._runtime(target, draft, 32)
rng = np.random.default_rng(0)
seq0 = [target.bos_id] + rng.integers(2, target.cfg.vocab, 127).tolist()
invt = 1.0
def timed(body, reps=3):
    rt.reset(seq0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(reps):
        s.record(); g.replay(); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts)
for gm in gammas:
    s0 = lambda: torch.cuda.current_stream()
    xs = lambda j: fastpath._addr(rt.chain, j)
    t_draft = timed(lambda: rt._draft_block(gm, 1, xs, invt, False, s0()))
    def tgt():
        _lib.check(rt.lib.pearl_llama_forward(target.handle, _device.ptr(rt.target_in), gm, rt._state_ptr(fastpath.S_TPOS),
                                              0, _device.ptr(rt.target_rows), _device.stream_ptr(s0())), "t")
    t_tgt = timed(tgt)
    t_post = timed(lambda: rt._pearl_body(gm - 1, gm, 1, invt, False, True))
    t_post_serial = timed(lambda: rt._pearl_body(gm - 1, gm, 1, invt, False, False))
    t_pre = timed(lambda: rt._pearl_body(0, gm, 1, invt, False, True))
    t_sd = timed(lambda: rt._sd_body(gm, 1, invt, False))
    print(f"gamma={gm:2d}: draft block {t_draft:.3f} ms | target M={gm} {t_tgt:.3f} ms | PEARL post {t_post:.3f} "
          f"(serial {t_post_serial:.3f}) pre {t_pre:.3f} | SD {t_sd:.3f} ms", flush=True)
