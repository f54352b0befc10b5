"""Rendezvous-timeout semantics (b2comm.h, b2_comm_set_timeout_ms): one rank
arrives long after the device timeout; no rank may return success for that
call or keep using the communicator afterwards.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29531 tests/mp_timeout.py

Rank 0 prints one JSON line; exit code 1 on any violation.
"""
from __future__ import annotations

import json
import os
import sys
import time
import traceback

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2107_01499_b200 as b2  # noqa: E402

U8 = b2.Codec(b2.CodecKind.uniform8)
TIMEOUT_MS = 400
LATE_S = 2.0


def attempt(fn):
    """-> 'ok' or the status name of the raised error"""
    try:
        fn()
        return "ok"
    except b2.Error as e:
        return "timeout" if getattr(e, "status", None) == b2._lib.B2_ERR_TIMEOUT else f"error:{e}"


def scenario(rank, world, dev, prim):
    ep = b2.B200Endpoint(rank, world, dev, timeout_ms=TIMEOUT_MS)
    n = 1_000_003
    x = torch.randn(n, device="cuda")
    topo = b2.Topology(b2.TopologyKind.ring, world, 0)

    def call():
        if prim == "c_lp_s":
            b2.c_lp_s(ep, 0.0, x, U8, None, bucket=7)
        elif prim == "d_lp_s":
            b2.d_lp_s(ep, 0.0, x, topo, 0, U8, b2.ReduceMode.average, bucket=7)
        else:
            b2.c_fp_s(ep, 0.0, x, bucket=7)

    res = {"warm": attempt(call)}  # both ranks on time: windows exist, epoch 1 done
    dist.barrier()
    if rank == world - 1:
        time.sleep(LATE_S)  # far beyond the device timeout
    res["late_call"] = attempt(call)
    dist.barrier()
    res["poisoned"] = ep.poisoned()
    res["next_call"] = attempt(call)  # everybody on time again: still refused
    res["sync"] = attempt(ep.sync)
    ep.close()
    # a fresh communicator works again
    ep2 = b2.B200Endpoint(rank, world, dev, timeout_ms=TIMEOUT_MS)
    y = torch.ones(4096, device="cuda")
    b2.c_fp_s(ep2, 0.0, y, bucket=8)
    res["fresh_ok"] = bool(torch.all(y == float(world)).item())
    ep2.close()
    return res


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    out, bad = {}, []
    for prim in ("c_lp_s", "d_lp_s", "c_fp_s"):
        try:
            r = scenario(rank, world, dev, prim)
        except Exception:
            r = {"exception": traceback.format_exc()[-800:]}
        out[prim] = r
        if r.get("warm") != "ok":
            bad.append(f"rank{rank} {prim}: warm-up call failed {r}")
        late = world - 1
        # D_LP_S over the ring: a rank that is not a neighbour of the late rank
        # never waits for it, and its (correct) result may stand
        depends = prim != "d_lp_s" or late in b2.Topology(b2.TopologyKind.ring, world, 0).neighbors(rank, 0)
        if depends and r.get("late_call") == "ok":
            bad.append(f"rank{rank} {prim}: the late call returned success")
        if r.get("next_call") != "timeout" or r.get("sync") != "timeout" or not r.get("poisoned", False):
            bad.append(f"rank{rank} {prim}: communicator kept working after the timeout {r}")
        if not r.get("fresh_ok", False):
            bad.append(f"rank{rank} {prim}: a fresh communicator does not work {r}")
        dist.barrier()
    allres = [None] * world
    dist.all_gather_object(allres, (out, bad))
    if rank == 0:
        fails = [b for _, bs in allres for b in bs]
        print(json.dumps({"world": world, "results": [o for o, _ in allres], "failed": len(fails),
                          "failures": fails}))
    ok = all(not bs for _, bs in allres)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
