"""Host-side cost of one primitive call (dev tool): per-call wall time of the
Python plumbing + C ABI launch on a tiny bucket (the GPU is never the bound),
against the raw ctypes call of the same entry point."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2107_01499_b200 as b2  # noqa: E402

ep = b2.B200Endpoint(0, 1, 0)
x = torch.randn(4096, device="cuda")
U8 = b2.Codec(b2.CodecKind.uniform8)
ring = b2.Topology(b2.TopologyKind.ring, 1, 0)
codes = torch.empty(4096 + 64, dtype=torch.uint8, device="cuda")
hdr = torch.empty(4, device="cuda")
N = 2000


def per_call(fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return round(1e6 * (t1 - t0) / N, 2), round(1e6 * (t2 - t0) / N, 2)


s = torch.cuda.current_stream().cuda_stream
h, p = ep.handle, x.data_ptr()
res = {
    "python c_lp_s": per_call(lambda: b2.c_lp_s(ep, 0.0, x, U8, None, blocking=False)),
    "ctypes b2_c_lp_s": per_call(lambda: b2.lib.b2_c_lp_s(h, p, 4096, 1, 0, 0, 0, 0, 0, s)),
    "python d_lp_s": per_call(lambda: b2.d_lp_s(ep, 0.0, x, ring, 0, U8, b2.ReduceMode.average, blocking=False)),
    "ctypes b2_u8_encode+decode": per_call(lambda: (b2.lib.b2_u8_encode(p, 4096, codes.data_ptr(), hdr.data_ptr(), s),
                                                   b2.lib.b2_u8_decode(codes.data_ptr(), hdr.data_ptr(), 4096, p, s))),
}
for k, (host, drain) in res.items():
    print(f"{k}: {host} us/call host, {drain} us/call incl. drain")
