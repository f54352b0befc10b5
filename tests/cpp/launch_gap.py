"""Per-call gap between back-to-back C_LP_S launches at g=1: device time of
20 calls bracketed by events, through (a) the Python API and (b) the C ABI
directly, vs the kernel time ncu reports (dev helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2107_01499_b200 as b2
from paper_2107_01499_b200._lib import lib

n = 100_000_000
ep = b2.B200Endpoint(0, 1, 0)
xs = [torch.rand(n, device="cuda") * 2 - 1 for _ in range(4)]
codec = b2.Codec(b2.CodecKind.uniform8)
s = torch.cuda.current_stream()
for i in range(5):
    b2.c_lp_s(ep, 0.0, xs[i % 4], codec, None, blocking=False)
torch.cuda.synchronize()
for mode in ("python", "cabi", "cabi-trace"):
    if mode == "cabi-trace":
        ep.enable_trace(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for i in range(20):
        if mode == "python":
            b2.c_lp_s(ep, 0.0, xs[i % 4], codec, None, blocking=False)
        else:
            lib.b2_c_lp_s(ep.handle, xs[i % 4].data_ptr(), n, 1, None, 0, None, 0, 0, s.cuda_stream)
    e1.record(s)
    t1 = time.perf_counter()
    e1.synchronize()
    print(f"{mode}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/call device, host enqueue {(t1 - t0) / 20 * 1e6:.1f} us/call")
    if mode == "cabi-trace":
        print(ep.read_trace())
        ep.enable_trace(False)
