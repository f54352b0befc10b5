"""Dev tool: per-CTA phase stamps of one c_lp_s call (torchrun, any world)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, torch.distributed as dist
import paper_2107_01499_b200 as b2
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(rank)
ep = b2.B200Endpoint(rank, world, rank)
n = int(os.environ.get("N", 100_000_000))
x = torch.empty(n, device="cuda")
b2.lib.b2_fill_synthetic(x.data_ptr(), n, 2026 + rank, 0, torch.cuda.current_stream().cuda_stream)
U8 = b2.Codec(b2.CodecKind.uniform8)
for _ in range(3):
    b2.c_lp_s(ep, 0.0, x, U8, None)
ep.enable_trace(True)
for it in range(3):
    dist.barrier(); torch.cuda.synchronize()
    b2.c_lp_s(ep, 0.0, x, U8, None)
    t = ep.read_trace(raw=True)
    names = ep.TRACE_POINTS
    raw0 = None
    out = {}
    for i, nm in enumerate(names):
        col = t[:, i]
        if np.all(np.isnan(col)):
            continue
        k = int(np.nanargmax(col))
        out[nm] = [round(float(np.nanmedian(col)), 1), round(float(np.nanmax(col)), 1), k]
    allv = [None] * world
    dist.all_gather_object(allv, out)
    if rank == 0:
        for r, o in enumerate(allv):
            print(it, r, json.dumps(o))
dist.destroy_process_group()
