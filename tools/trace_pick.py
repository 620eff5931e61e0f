"""Phase timeline of the pick kernel (build/trace/libpearl_trace.so, -DPEARL_TRACE_PICK).

    PEARL_LIB_PATH=build/trace/libpearl_trace.so python tools/trace_pick.py [V]
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_11850_b200 import _lib, _device
V = int(sys.argv[1]) if len(sys.argv) > 1 else 32000
lib = _lib.load()
lib.pearl_debug_trace.argtypes = [ctypes.c_void_p]
_lib.prepare_vocab(V)
dev = torch.device("cuda")
logits = torch.randn(V, device=dev) * 3
rows = _device.row_ptrs([logits], dev)
u = torch.rand(4096, dtype=torch.float64, device=dev)
cur = torch.zeros(1, dtype=torch.int32, device=dev)
out = torch.zeros(4, dtype=torch.int32, device=dev)
st = torch.zeros(1, dtype=torch.int32, device=dev)
work = torch.zeros(int(lib.pearl_verify_work_bytes(4)), dtype=torch.uint8, device=dev)
for greedy in (0, 1):
    for rep in range(5):
        _lib.check(lib.pearl_sample_rows(1, _device.ptr(rows), 1, V, _device.ptr(u), 4096, _device.ptr(cur), 1.0,
                                         (_lib.F_GREEDY if greedy else 0), _device.ptr(out), None, _device.ptr(st),
                                         _device.ptr(work), _device.stream_ptr()), "pick")
        torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 32)()
    lib.pearl_debug_trace(buf)
    t0 = buf[0]
    print("greedy" if greedy else "sampled", {k: buf[k] - t0 for k in range(32) if buf[k] >= t0 and buf[k] - t0 < 10**7})
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for rep in range(50):
        lib.pearl_sample_rows(1, _device.ptr(rows), 1, V, _device.ptr(u), 4096, _device.ptr(cur), 1.0,
                              (_lib.F_GREEDY if greedy else 0), _device.ptr(out), None, _device.ptr(st),
                              _device.ptr(work), _device.stream_ptr())
    e.record(); e.synchronize()
    print("  back-to-back eager us/pick:", s.elapsed_time(e) / 50 * 1e3)
