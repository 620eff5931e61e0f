"""Run one eager draft block (gamma tokens) of the 7B/68M runtime (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_11850_b200 import llama, fastpath
gm = int(sys.argv[1]) if len(sys.argv) > 1 else 4
D = int(os.environ.get("PEARL_DRAFT_SMS", "0"))  # > 0: run the block on the draft's green partition
target, draft = llama.build_pair("llama2-7b/68m", gemm_target="tcgen05", align=llama.AlignSpec(branch_std=5e-4),
                                 max_seq=400, max_tokens=64, draft_sms=D)
rt = fastpath._runtime(target, draft, 32)
rng = np.random.default_rng(0)
seq0 = [target.bos_id] + rng.integers(2, target.cfg.vocab, 127).tolist()
rt.reset(seq0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("draft_block")
st = rt.draft_stream if D > 0 else torch.cuda.current_stream()
with torch.cuda.stream(st):
    rt._draft_block(gm, 1, lambda j: fastpath._addr(rt.chain, j), 1.0, False, st)
torch.cuda.synchronize()
print("done")
