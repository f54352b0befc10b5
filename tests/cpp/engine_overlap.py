"""Bucketed C_LP_S overlapping a synthetic VGG16 backward.

Backward is simulated on the compute stream (torch.cuda._sleep per layer,
proportional to the layer's parameter count); gradients are the VGG16 layer
shapes (138.36M parameters), bucketed by the engine's greedy reverse-order
packing (8 MiB default).  Reports, max over ranks:
  backward only | backward then every bucket (serial) | engine overlap.

  python -m torch.distributed.run --nproc-per-node G tests/cpp/engine_overlap.py [backward_ms] [capacity_MiB]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import torch.distributed as dist
import paper_2107_01499_b200 as b2
from paper_2107_01499_b200.engine import OverlapEngine

VGG16 = [1792, 36928, 73856, 147584, 295168, 590080, 590080, 1180160, 2359808, 2359808, 2359808, 2359808,
         2359808, 102764544, 16781312, 4097000]

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
backward_ms = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
cap = int(float(sys.argv[2]) * (1 << 20)) if len(sys.argv) > 2 else 8 << 20
ep = b2.B200Endpoint(rank, world, dev)
eng = OverlapEngine(ep, VGG16, capacity_bytes=cap)
total = sum(VGG16)
cycles_per_param = backward_ms * 1e-3 * 1.9e9 / total  # ~SM clock
for layer, n in enumerate(VGG16):
    eng.grad(layer).uniform_(-2 ** -10, 2 ** -10)


def backward(overlap: bool, comm: bool):
    s = torch.cuda.current_stream()
    for layer in reversed(range(len(VGG16))):
        torch.cuda._sleep(int(cycles_per_param * VGG16[layer]) + 1)
        if comm and overlap:
            eng.layer_done(layer)
    if comm and not overlap:
        for layer in reversed(range(len(VGG16))):
            eng.layer_done(layer)
    if comm:
        eng.finish()


def timed(overlap, comm, iters=10):
    for _ in range(3):
        backward(overlap, comm)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        backward(overlap, comm)
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


t_bwd = timed(False, False)
t_serial = timed(False, True)
t_overlap = timed(True, True)
comm = t_serial - t_bwd
if rank == 0:
    print(json.dumps({"world": world, "params": total, "buckets": len(eng.buckets), "capacity_MiB": cap / 2 ** 20,
                      "backward_ms": round(t_bwd, 3), "serial_ms": round(t_serial, 3),
                      "overlap_ms": round(t_overlap, 3), "comm_ms": round(comm, 3),
                      "hidden_frac": round((t_serial - t_overlap) / comm, 3) if comm > 0 else None}))
ep.close()
dist.destroy_process_group()
