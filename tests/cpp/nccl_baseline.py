"""NCCL full-precision baseline beside C_FP_S (north_star: NCCL only for the
full-precision baselines).  torch.distributed all_reduce(SUM) of N fp32 per
rank over NCCL vs b2 c_fp_s on the same buffers; device time per call, max
over ranks.  NCCL's ring/NVLS reduction order differs from the reference's
ascending-rank fp64 fold, so it is a speed baseline, not a drop-in.

  python -m torch.distributed.run --nproc-per-node G tests/cpp/nccl_baseline.py [N]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import torch.distributed as dist
import paper_2107_01499_b200 as b2

dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_000_000
xs = [torch.rand(n, device="cuda") * 2 ** -8 for _ in range(8)]
ep = b2.B200Endpoint(rank, world, dev)


def timed(fn, steps=50):
    for i in range(5):
        fn(xs[i % 8])
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        fn(xs[i % 8])
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


t_nccl = timed(lambda x: dist.all_reduce(x))
t_b2 = timed(lambda x: b2.c_fp_s(ep, 0.0, x, blocking=False))
if rank == 0:
    print(json.dumps({"n": n, "world": world, "nccl_allreduce_ms": round(t_nccl, 4),
                      "b2_c_fp_s_ms": round(t_b2, 4),
                      "nccl_busbw_gbs": round(2 * (world - 1) / world * 4 * n / (t_nccl / 1e3) / 1e9, 1),
                      "b2_busbw_gbs": round(2 * (world - 1) / world * 4 * n / (t_b2 / 1e3) / 1e9, 1)}))
ep.close()
dist.destroy_process_group()
