"""Measure logits error of the CUDA forward vs oracle/llama.py at the BASELINE
shapes (reduced depth, full width) -- the numbers the stated tolerances in
tests/test_parity_shapes_gpu.py are set from.

    python tools/parity_probe.py [pair ...]
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.llama import OracleLlama  # noqa: E402
from paper_2408_11850_b200 import llama  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False

PAIRS = {"llama2-7b/68m": (2, 2), "dsc-33b/1.3b": (2, 2), "llama3-70b/8b": (2, 2)}


def probe(pair, depth, n_tok=200, branch_std=0.02, gemm_target="tcgen05"):
    tgt, drf = llama.build_pair(pair, depth=depth, max_seq=512, max_tokens=128, gemm_target=gemm_target,
                                align=llama.AlignSpec(branch_std=branch_std))
    out = {}
    rng = np.random.default_rng(0)
    for m in (tgt, drf):
        toks = [m.bos_id] + rng.integers(0, m.cfg.vocab, n_tok - 1).tolist()
        got = m.forward_logits(toks)
        row = {"gemm": m.gemm, "hd": m.cfg.head_dim, "H": m.cfg.n_heads, "KV": m.cfg.n_kv_heads,
               "theta": m.cfg.rope_theta, "V": m.cfg.vocab}
        for name, b in (("bf16pts", True), ("fp32", False)):
            o = OracleLlama(m.cfg, m.w, device="cuda", bf16_points=b, max_seq=512, norm_fold=m.gemm == "tcgen05")
            want = o.forward(toks, 0)
            del o
            err = (got - want).abs()
            scale = want.abs().amax(-1, keepdim=True)
            top2 = want.topk(2, -1).values
            row[name] = {"max_abs": float(err.max()), "max_rel_rowmax": float((err / scale).max()),
                         "p999_abs": float(err.flatten().kthvalue(int(0.999 * err.numel())).values),
                         "logit_absmax": float(want.abs().max()),
                         "argmax_agree": float((got.argmax(-1) == want.argmax(-1)).float().mean()),
                         "min_margin": float((top2[:, 0] - top2[:, 1]).min())}
            torch.cuda.empty_cache()
        out[m.cfg.name] = row
    del tgt, drf
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if "/" in a] or list(PAIRS)
    bstd = float(os.environ.get("BRANCH_STD", "0.02"))
    res = {}
    for p in names:
        for gt in ("tcgen05", "cudacore"):
            res[f"{p}:{gt}"] = r = probe(p, PAIRS[p], branch_std=bstd, gemm_target=gt)
            print(p, gt, json.dumps({m: {k: v for k, v in row.items() if k in ("gemm", "bf16pts", "fp32")}
                                     for m, row in r.items()}), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/parity_probe.json", "w") as fh:
        json.dump(res, fh, indent=1)
