import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2408_11850_b200 import llama
t, d = llama.build_pair("llama2-7b/68m", gemm_target="tcgen05", align=llama.AlignSpec(branch_std=5e-4), max_seq=400, max_tokens=64, l2_draft=True, draft_sms=40)
print("draft l2 granted", d.l2_granted, "persisting max", torch.cuda.get_device_properties(0).L2_cache_size if hasattr(torch.cuda.get_device_properties(0), "L2_cache_size") else None)
