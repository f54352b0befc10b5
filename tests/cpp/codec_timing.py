"""Dev tool: in-stream time of the 4M codec kernels (graphs of K back-to-back
launches, so the graph launch is amortised): encode alone, decode alone, the
pair -- what a step of `bench.py --prim codec` is made of."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2107_01499_b200 as b2  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
K = 20
x = torch.empty(n, device="cuda")
b2.lib.b2_fill_synthetic(x.data_ptr(), n, 2026, 0, torch.cuda.current_stream().cuda_stream)
codes = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
hdr = torch.empty(4, device="cuda")


def enc():
    s = torch.cuda.current_stream().cuda_stream
    b2._lib.check(b2.lib.b2_u8_encode(x.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(), s))


def dec():
    s = torch.cuda.current_stream().cuda_stream
    b2._lib.check(b2.lib.b2_u8_decode(codes.data_ptr(), hdr.data_ptr(), n, x.data_ptr(), s))


def both():
    enc()
    dec()


res = {}
for name, fn in (("encode", enc), ("decode", dec), ("encode+decode", both)):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            for _ in range(K):
                fn()
    torch.cuda.current_stream().wait_stream(cap)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    e1.synchronize()
    res[name] = round(e0.elapsed_time(e1) * 1e3 / (10 * K), 2)
print(json.dumps({"n": n, "us_per_call_in_graph": res}))
