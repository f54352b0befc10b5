"""PCIe ceiling for bench.py's e2e leg: pinned host <-> device copies of one
100M-fp32 bucket (400 MB), H2D alone, D2H alone and both at once on two
streams (what the e2e pipeline overlaps).  Prints one JSON line.

    python tests/cpp/pcie_probe.py [--mb 400] [--reps 5]
"""
import argparse
import json

import torch


def timed(fn, reps, streams):
    for s in streams:
        s.synchronize()
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(streams[0])
        for s in streams[1:]:
            s.wait_event(e0)
        fn()
        for s in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            streams[0].wait_event(ev)
        e1.record(streams[0])
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=400)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    nbytes = a.mb * 1_000_000
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h2d = timed(h2d, a.reps, [s1])
    t_d2h = timed(d2h, a.reps, [s2])
    t_both = timed(both, a.reps, [s1, s2])
    gb = nbytes / 1e9
    print(json.dumps({
        "probe": "pcie pinned copies", "bytes": nbytes,
        "h2d_GBps": round(gb / t_h2d, 2), "d2h_GBps": round(gb / t_d2h, 2),
        "both_ms": round(t_both * 1e3, 3),
        "both_each_dir_GBps": round(gb / t_both, 2),
    }))


if __name__ == "__main__":
    main()
