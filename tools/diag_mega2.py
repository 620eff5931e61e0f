"""Diagnostics: first diverging phase between the persistent and per-op forward."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_11850_b200 import llama, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 16
target, _ = llama.build_pair(name, gemm_target="tcgen05", max_seq=512, max_tokens=32)
c = target.cfg
V = c.vocab
rng = np.random.default_rng(7)
prefix = [target.bos_id] + rng.integers(0, V, 20).tolist()
P = len(prefix)
win = rng.integers(0, V, M).tolist()
T = 32
bufs = {"h": (0, torch.float32, c.d_model), "x": (1, torch.bfloat16, c.d_model), "q": (2, torch.bfloat16, c.n_heads * c.head_dim),
        "o": (3, torch.bfloat16, c.n_heads * c.head_dim), "act": (4, torch.bfloat16, c.ffn)}
names = ["embed", "norm1", "qkv", "attn", "o", "norm2", "gate_up", "down", "norm1'", "qkv'", "attn'"]
for stop in range(1, 12):
    got = {}
    for flags in (4, 0, 4 + 100, 0 + 100):  # persistent, per-op (x2)
        os.environ.pop("PEARL_STOP", None)
        target.forward_logits(prefix)
        for k, (w, dt, n) in bufs.items():   # poison
            pass
        pos = torch.tensor([P], dtype=torch.int32, device="cuda")
        t = torch.tensor(win, dtype=torch.int32, device="cuda")
        os.environ["PEARL_STOP"] = str(stop)
        target.forward(t, M, pos, flags % 100, None)
        os.environ.pop("PEARL_STOP", None)
        torch.cuda.synchronize()
        out = {}
        for k, (w, dt, n) in bufs.items():
            b = torch.empty(M, n, dtype=dt, device="cuda")
            _lib.check(_lib.load().pearl_llama_debug_buffer(target.handle, w, b.data_ptr(), b.numel() * b.element_size(),
                                                            None), "dbg")
            out[k] = b
        torch.cuda.synchronize()
        got[flags] = out
    dd = lambda a, b: {k: f"{float((got[a][k].float() - got[b][k].float()).abs().max()):.1e}" for k in bufs}
    print(f"after {names[stop-1]:8s}: mega-perop {dd(4, 0)} | mega-mega {dd(4, 104)} | perop-perop {dd(0, 100)}", flush=True)
