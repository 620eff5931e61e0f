"""Which elements of h differ after the O projection (persistent vs per-op)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_11850_b200 import llama, _lib
M = int(sys.argv[1]) if len(sys.argv) > 1 else 4
stop = int(sys.argv[2]) if len(sys.argv) > 2 else 5
target, _ = llama.build_pair("tiny", gemm_target="tcgen05", max_seq=512, max_tokens=32)
c = target.cfg
V = c.vocab
rng = np.random.default_rng(7)
prefix = [target.bos_id] + rng.integers(0, V, 20).tolist()
P = len(prefix)
win = rng.integers(0, V, M).tolist()
def run(flags, stop):
    os.environ.pop("PEARL_STOP", None)
    target.forward_logits(prefix)
    pos = torch.tensor([P], dtype=torch.int32, device="cuda")
    t = torch.tensor(win, dtype=torch.int32, device="cuda")
    os.environ["PEARL_STOP"] = str(stop)
    target.forward(t, M, pos, flags, None)
    os.environ.pop("PEARL_STOP", None)
    torch.cuda.synchronize()
    outs = []
    for w, dt, n in ((0, torch.float32, c.d_model), (3, torch.bfloat16, c.n_heads * c.head_dim), (4, torch.bfloat16, c.ffn),
                     (1, torch.bfloat16, c.d_model), (2, torch.bfloat16, c.n_heads * c.head_dim)):
        b = torch.empty(M, n, dtype=dt, device="cuda")
        _lib.check(_lib.load().pearl_llama_debug_buffer(target.handle, w, b.data_ptr(), b.numel() * b.element_size(), None), "d")
        outs.append(b)
    fl = torch.empty(64, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().pearl_llama_debug_buffer(target.handle, 5, fl.data_ptr(), 256, None), "d")
    ct = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().pearl_llama_debug_buffer(target.handle, 6, ct.data_ptr(), 4, None), "d")
    torch.cuda.synchronize()
    print(f"  flags={flags} stop={stop}: tile_flags nonzero at {fl.nonzero().flatten().tolist()} counter={ct.item() (first phase counter; 0 between launches)}")
    return outs
h0, o0, _, x0, q0 = run(4, stop - 1)
_, ostale, _, _, _ = run(4, stop - 2)
hm, om, am, _, _ = run(4, stop)
hp, op, ap, _, _ = run(0, stop)
W = target.w["layers"][0]["wo"] if isinstance(target.w, dict) and "layers" in target.w else None
print("o equal before:", torch.equal(om, op), " mega h unchanged by O:", torch.equal(hm, h0))
d = (hm - hp).abs()
bad = (d > 0).nonzero()
print("n differing:", bad.shape[0], "of", d.numel())
rows = sorted(set(bad[:, 0].tolist())); cols = bad[:, 1]
print("rows:", rows, "col tiles:", sorted(set((cols // 128).tolist())), "cols sample:", cols[:20].tolist())
wo = target.w["layers"][0]["wo"].double()
ref = h0.double() + om.double() @ wo.T
print("max |mega-ref| =", float((hm.double() - ref).abs().max()), " max |perop-ref| =", float((hp.double() - ref).abs().max()))
print("per-row max |mega-perop|:", [float(d[r].max()) for r in range(M)])
for name, X in (("o", om), ("o_stale", ostale), ("x", x0), ("q", q0), ("zeros", torch.zeros_like(om))):
    r = h0.double() + X.double() @ wo.T
    print(f"candidate X={name}: max |mega - h0 - X wo^T| = {float((hm.double() - r).abs().max()):.3e}")
for s in range(4):
    r = h0.double() + om[s:s+1].double().expand(M, -1) @ wo.T
    print(f"candidate X=row{s} broadcast: {float((hm.double() - r).abs().max()):.3e}")
