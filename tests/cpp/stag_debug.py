"""Dev tool: back-to-back C_LP_S calls with tracing and a short device
timeout; on a rendezvous timeout prints, per rank, how far every CTA got
(trace points of the failing launch, microseconds after its first CTA).

    torchrun --nproc-per-node G tests/cpp/stag_debug.py <elements> <calls> [nbuf]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2107_01499_b200 as b2  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
n = int(sys.argv[1])
calls = int(sys.argv[2])
nbuf = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ep = b2.B200Endpoint(rank, world, dev, timeout_ms=5000)
ep.enable_trace(True)
U8 = b2.Codec(b2.CodecKind.uniform8)
xs = [torch.empty(n, device="cuda") for _ in range(nbuf)]
for i, x in enumerate(xs):
    b2.lib.b2_fill_synthetic(x.data_ptr(), n, 2026 + rank + 10 * i, 0, torch.cuda.current_stream().cuda_stream)
    x.mul_(2.0 ** -20)
status = "ok"
failed_at = None
for c in range(calls):
    try:
        b2.c_lp_s(ep, 0.0, xs[c % nbuf], U8, None, blocking=True)
    except b2.Error as e:
        status, failed_at = str(e), c
        break
tr = ep.read_trace(raw=True)
names = b2.B200Endpoint.TRACE_POINTS
out = {"rank": rank, "status": status, "failed_at": failed_at}
if failed_at is not None:
    # per point: how many CTAs reached it, and the max time
    out["points"] = {names[i]: [int(np.sum(~np.isnan(tr[:, i]))), float(np.nanmax(tr[:, i])) if np.any(~np.isnan(tr[:, i])) else None]
                     for i in range(len(names))}
allv = [None] * world
dist.all_gather_object(allv, out)
if rank == 0:
    for v in allv:
        print(json.dumps(v))
dist.barrier()
dist.destroy_process_group()
