"""Bucketed C_LP_S overlapping a REAL backward (SURVEY.md 8f rank 1,
engine.cpp:113-153): every VGG16 layer's backward is a bf16 GEMM on the
compute stream (cuBLAS), sized so that its FLOPs are proportional to the
layer's parameter count and the whole backward takes ~backward_ms; the
gradients (VGG16 layer shapes, 138.36M parameters) go through the engine's
greedy reverse-order buckets.  The communication kernels compete with the
GEMMs for SMs; the SM budget (b2_comm_set_sm_budget) decides how many SMs a
primitive takes.  Per budget, max over ranks:

  backward_ms  GEMMs only
  comm_ms      every bucket back to back, no compute
  overlap_ms   GEMMs with each bucket issued at its trigger layer
  hidden_frac  (backward + comm - overlap) / comm

  python -m torch.distributed.run --nproc-per-node G tests/cpp/engine_overlap.py \
      [backward_ms=5] [capacity_MiB=25] [budgets=0,74,32,16]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2107_01499_b200 as b2  # noqa: E402
from paper_2107_01499_b200.engine import OverlapEngine  # noqa: E402

VGG16 = [1792, 36928, 73856, 147584, 295168, 590080, 590080, 1180160, 2359808, 2359808, 2359808, 2359808,
         2359808, 102764544, 16781312, 4097000]

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
backward_ms = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
cap = int(float(sys.argv[2]) * (1 << 20)) if len(sys.argv) > 2 else 25 << 20
budgets = [int(b) for b in (sys.argv[3] if len(sys.argv) > 3 else "0,74,32,16").split(",")]
total = sum(VGG16)

K = 4096
W = torch.randn(K, K, device="cuda", dtype=torch.bfloat16)
A = torch.randn(1 << 18, K, device="cuda", dtype=torch.bfloat16)
# rows per layer: FLOPs proportional to parameters, calibrated to backward_ms
torch.matmul(A[:8192], W)
torch.cuda.synchronize()
c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
c0.record()
for _ in range(10):
    torch.matmul(A[:65536], W)
c1.record()
c1.synchronize()
ms_per_row = c0.elapsed_time(c1) / 10 / 65536
rows_total = backward_ms / ms_per_row
ROWS = [max(128, int(rows_total * n / total) // 128 * 128) for n in VGG16]
ROWS = [min(r, A.shape[0]) for r in ROWS]


def backward(eng, overlap: bool, comm: bool):
    for layer in reversed(range(len(VGG16))):
        torch.matmul(A[:ROWS[layer]], W)  # this layer's backward GEMM
        if comm and overlap:
            eng.layer_done(layer)
    if comm and not overlap:
        for layer in reversed(range(len(VGG16))):
            eng.layer_done(layer)
    if comm:
        eng.finish()


def comm_only(eng):
    for layer in reversed(range(len(VGG16))):
        eng.layer_done(layer)
    eng.finish()


def timed(fn, iters=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


t_bwd = timed(lambda: backward(None, False, False))
for k in budgets:
    ep = b2.B200Endpoint(rank, world, dev)
    eng = OverlapEngine(ep, VGG16, capacity_bytes=cap, sm_budget=k)
    for layer in range(len(VGG16)):
        eng.grad(layer).uniform_(-2 ** -10, 2 ** -10)
    t_comm = timed(lambda: comm_only(eng))
    t_over = timed(lambda: backward(eng, True, True))
    eng.synchronize()
    if rank == 0:
        print(json.dumps({"world": world, "sm_budget": k or torch.cuda.get_device_properties(dev).multi_processor_count,
                          "params": total, "buckets": len(eng.buckets), "capacity_MiB": cap / 2 ** 20,
                          "backward": "bf16 GEMMs [rows x 4096] @ [4096 x 4096], rows proportional to the layer",
                          "backward_ms": round(t_bwd, 3), "comm_ms": round(t_comm, 3),
                          "overlap_ms": round(t_over, 3),
                          "hidden_frac": round((t_bwd + t_comm - t_over) / t_comm, 3) if t_comm > 0 else None}),
              flush=True)
    del eng
    ep.close()
dist.barrier()
dist.destroy_process_group()
