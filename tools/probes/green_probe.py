"""Probe: green contexts (SM partitions) + torch streams + CUDA-graph capture."""
import torch, time
from cuda.bindings import driver as d

def ck(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    assert err == d.CUresult.CUDA_SUCCESS, err
    return rest[0] if len(rest) == 1 else rest

torch.cuda.init()
x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
ck(d.cuInit(0))
dev = ck(d.cuDeviceGet(0))
res = ck(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
print("SMs:", res.sm.smCount)
out = ck(d.cuDevSmResourceSplitByCount(1, res, 0, 16))
print("split ->", out[1] if len(out) > 1 else out)
groups, n, remaining = out
g0 = groups[0]
print("group0 SMs", g0.sm.smCount, "remaining", remaining.sm.smCount)
def mkstream(r):
    desc = ck(d.cuDevResourceGenerateDesc([r], 1))
    gctx = ck(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    st = ck(d.cuGreenCtxStreamCreate(gctx, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    return gctx, st
gs, ss = mkstream(g0)
gt, st = mkstream(remaining)
small = torch.cuda.ExternalStream(int(st and ss))
s_small = torch.cuda.ExternalStream(int(ss))
s_big = torch.cuda.ExternalStream(int(st))
def t_mm(stream, n=5):
    with torch.cuda.stream(stream):
        y = x @ x
        stream.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(stream)
        for _ in range(n):
            y = x @ x
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / n
print("matmul ms: default %.3f | green16 %.3f | green-rest %.3f" % (t_mm(torch.cuda.current_stream()), t_mm(s_small), t_mm(s_big)))
# graph capture with a fork into both green streams
g = torch.cuda.CUDAGraph()
a = torch.empty_like(x); b = torch.empty_like(x)
try:
    with torch.cuda.graph(g):
        s0 = torch.cuda.current_stream()
        s_small.wait_stream(s0); s_big.wait_stream(s0)
        with torch.cuda.stream(s_small):
            torch.matmul(x, x, out=a)
        with torch.cuda.stream(s_big):
            torch.matmul(x, x, out=b)
        s0.wait_stream(s_small); s0.wait_stream(s_big)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); e1.synchronize()
    print("graph replay ok: %.3f ms; results equal:" % e0.elapsed_time(e1), torch.equal(a, b), torch.equal(a, x @ x))
except Exception as ex:
    print("graph capture failed:", repr(ex)[:300])
