"""Draft block time on the green-context draft partition: alone, and while the
target forward runs on the rest (PEARL_DRAFT_SMS sets the partition)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2408_11850_b200 import llama, fastpath, _lib, _device
D = int(os.environ.get("PEARL_DRAFT_SMS", "40"))
target, draft = llama.build_pair("llama2-7b/68m", gemm_target="tcgen05", align=llama.AlignSpec(branch_std=5e-4),
                                 max_seq=600, max_tokens=64, draft_sms=D)
rt = fastpath._runtime(target, draft, 32)
seq0 = [target.bos_id] + np.random.default_rng(0).integers(2, 32000, 127).tolist()
ds, ts = rt.draft_stream, rt.target_stream
def timed(body, reps=3):
    rt.reset(seq0)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    out = []
    for _ in range(reps):
        s.record(); g.replay(); e.record(); e.synchronize(); out.append(s.elapsed_time(e))
    return min(out)
xs = lambda j: fastpath._addr(rt.chain, j)
for gm in (1, 8, 16, 24):
    def dblock():
        s0 = torch.cuda.current_stream()
        ds.wait_stream(s0)
        with torch.cuda.stream(ds):
            rt._draft_block(gm, 1, xs, 1.0, False, ds)
        s0.wait_stream(ds)
    def both():
        s0 = torch.cuda.current_stream()
        ds.wait_stream(s0); ts.wait_stream(s0)
        with torch.cuda.stream(ds):
            rt._draft_block(gm, 1, xs, 1.0, False, ds)
        with torch.cuda.stream(ts):
            _lib.check(rt.lib.pearl_llama_forward(target.handle, _device.ptr(rt.target_in), max(gm, 1), rt._state_ptr(fastpath.S_TPOS), 0, _device.ptr(rt.target_rows), _device.stream_ptr(ts)), "t")
        s0.wait_stream(ds); s0.wait_stream(ts)
    def tonly():
        s0 = torch.cuda.current_stream()
        ts.wait_stream(s0)
        with torch.cuda.stream(ts):
            _lib.check(rt.lib.pearl_llama_forward(target.handle, _device.ptr(rt.target_in), max(gm, 1), rt._state_ptr(fastpath.S_TPOS), 0, _device.ptr(rt.target_rows), _device.stream_ptr(ts)), "t")
        s0.wait_stream(ts)
    print(f"D={D} gamma={gm}: draft block alone on partition {timed(dblock):.3f} ms | target alone {timed(tonly):.3f} | both {timed(both):.3f} ms", flush=True)
