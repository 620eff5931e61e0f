"""Draft single-token forward time (CUDA graph) and 7B/68M step anatomy; run
twice with PEARL_GEMV1=0 / 1 for the K2 single-token A/B."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import llama
pair = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b/68m"
D = int(os.environ.get("PEARL_DRAFT_SMS", "0"))
target, draft = llama.build_pair(pair, gemm_target="tcgen05", align=llama.AlignSpec(branch_std=5e-4),
                                 max_seq=600, max_tokens=64, draft_sms=D)
ts = sorted(draft.measure_forward_time(1, iters=20) for _ in range(5))
print(f"{pair} GEMV1={os.environ.get('PEARL_GEMV1', '1')} draft_sms={D}: draft token forward "
      f"{ts[0]*1e6:.1f} us (median {ts[2]*1e6:.1f})", flush=True)
