"""Host-side cost of one c_lp_s call (dev tool): per-call wall time of the
Python plumbing + C ABI launch, on a tiny bucket so the GPU is never the bound."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2107_01499_b200 as b2
ep = b2.B200Endpoint(0, 1, 0)
x = torch.randn(4096, device="cuda")
U8 = b2.Codec(b2.CodecKind.uniform8)
for _ in range(10):
    b2.c_lp_s(ep, 0.0, x, U8, None, blocking=False)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    b2.c_lp_s(ep, 0.0, x, U8, None, blocking=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"python c_lp_s: {1e6*(t1-t0)/N:.1f} us/call host, {1e6*(t2-t0)/N:.1f} us/call incl. drain")
import ctypes as C
h = ep.handle; s = torch.cuda.current_stream().cuda_stream; p = x.data_ptr()
t0 = time.perf_counter()
for _ in range(N):
    b2.lib.b2_c_lp_s(h, p, 4096, 1, 0, 0, 0, 0, 0, s)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"raw ctypes b2_c_lp_s: {1e6*(t1-t0)/N:.1f} us/call host")
