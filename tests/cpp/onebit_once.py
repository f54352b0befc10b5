"""Three blocking C_LP_S onebit calls over a 100M-element bucket on one GPU
(the ncu capture target for onebit_central_kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2107_01499_b200 as b2  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ec = len(sys.argv) > 2 and sys.argv[2] == "ec"
ep = b2.B200Endpoint(0, 1, 0)
x = torch.empty(n, device="cuda")
b2.lib.b2_fill_synthetic(x.data_ptr(), n, 2026, 0, torch.cuda.current_stream().cuda_stream)
es = b2.ErrorState(n, n) if ec else None
for _ in range(3):
    b2.c_lp_s(ep, 0.0, x, b2.Codec(b2.CodecKind.onebit), es)
print("ok", float(x[:4].abs().sum()))
