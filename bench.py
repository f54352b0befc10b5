#!/usr/bin/env python3
"""Benchmark: C_LP_S (ByteGrad / MinMaxUInt8) allreduce of a 100M-element fp32
gradient bucket per GPU -- BASELINE.json's metric "effective gradient GB/s for
C_LP_S allreduce at 1/2/4/8 B200 vs roofline".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...           (N > 1)

A step is one c_lp_s call over the rank's resident 100M-element bucket (one
fused cooperative kernel launch per step).  Inputs are deterministic synthetic
gradients (splitmix64 hash, seed 2026 + rank) of 400 MB per GPU -- larger
than the 126 MB L2, so no flush is needed between steps.  Each step consumes
the previous step's output (always finite, the codec range never degenerates).

value     = whole-job effective gradient GB/s = N_gpus * 4 * elements / t_step
            (the per-GPU figure, BASELINE.md's definition 4N/wall, is
            config.per_gpu_gbs)
e2e       = same metric through the reference-facing API with HOST buffers:
            pinned H2D copy of the bucket, c_lp_s, D2H copy of the result, per step
roofline  = algorithmic bytes of the dominant (only) kernel / its event time,
            against MEASURED_PEAKS.json HBM copy bandwidth (g <= 4) or the
            measured 770 GB/s NVLink peer bandwidth (g = 8) -- see DESIGN.md 5
cpu_baseline = the unmodified reference (oracle/_ref) C_LP_S on this host's
            cores, one thread per worker, on a bounded sample (rank 0, N=1)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_ELEMS = 100_000_000
HBM_FALLBACK_GBS = 6650.0
NVL_PEER_GBS = 770.0   # measured peer copy, B200_PROFILING.md
NVL_NOMINAL_GBS = 900.0


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


PRIMS = {  # name -> (default elements, reference time_primitive id, metric label)
    "c_lp_s": (100_000_000, 2, "C_LP_S allreduce"),
    "c_fp_s": (25_000_000, 1, "C_FP_S allreduce"),
    "d_fp_s": (25_000_000, 3, "D_FP_S ring averaging"),
    "d_lp_s": (25_000_000, 4, "D_LP_S ring averaging"),
    "codec": (4_000_000, 0, "MinMaxUInt8 compress+decompress"),
    "onebit": (4_000_000, 5, "Onebit compress+decompress"),
    "c_lp_s_onebit": (100_000_000, 6, "C_LP_S onebit allreduce"),
    "d_lp_s_onebit": (25_000_000, 7, "D_LP_S onebit ring averaging"),
}


def ring_nbrs(g: int) -> int:
    """|N(i)| of the ring topology, self included (collectives.cpp:187-192)."""
    return min(g, 3)


def algorithmic_bytes(prim: str, n: int, g: int):
    """Per-GPU algorithmic (HBM, NVLink-ingress) bytes, SURVEY.md 8d."""
    nb = ring_nbrs(g)
    if prim == "c_lp_s":
        return 11 * n + n // g, 2 * n * (g - 1) // g
    if prim == "c_fp_s":
        if g == 1:  # collectives.cpp:49: one worker returns x untouched -- no device work at all
            return 0, 0
        return 4 * n + 4 * n // g + 8 * n * (g - 1) // g, 8 * n * (g - 1) // g
    if prim == "d_fp_s":
        return 4 * n * nb + 4 * n, 4 * n * (nb - 1)
    if prim == "d_lp_s":
        return 4 * n + n + n * nb + 4 * n, n * (nb - 1)
    if prim == "c_lp_s_onebit":  # x 4N; bits N/8 out, N/8 folded, N/8g second bits, N/8 gathered; x' 4N
        return 8 * n + 3 * n // 8 + n // (8 * g), n * (g - 1) // (4 * g)
    if prim == "d_lp_s_onebit":  # x 4N; my bits N/8; |N| neighbours' bits; x' 4N
        return 8 * n + (nb + 1) * n // 8, (nb - 1) * n // 8
    if prim == "onebit":  # read x, write bits, read bits, write x
        return 8 * n + 2 * ((n + 7) // 8), 0
    return 10 * n, 0  # codec: read x, write codes, read codes, write x


def kernel_label(prim: str, n: int, g: int) -> str:
    """The kernel a step launches (the library's dispatch: comm.cu central /
    decentral, codec.cu small_encode)."""
    if prim in ("c_lp_s", "c_fp_s"):
        cod = "uint8" if prim == "c_lp_s" else "identity"
        if g > 1 and n <= 4_000_000:
            return f"central_small_kernel<{cod}, g={g}> (register-resident, one cooperative launch per step)"
        if prim == "c_lp_s" and g == 2 and n % 32 == 0:
            return "central_stag_kernel<uint8> (staggered schedule, one cooperative launch per step)"
        return f"central_kernel<{cod}> (one fused launch per step)"
    if prim in ("d_lp_s", "d_fp_s"):
        cod = "uint8" if prim == "d_lp_s" else "identity"
        if n <= 16_000_000:
            return f"decent_small_kernel / decent_stream_kernel<{cod}> (per-CTA hand-off, one launch per step)"
        return f"decent_kernel<{cod}> (one fused launch per step)"
    return {"c_lp_s_onebit": "onebit_central_kernel<g, false> (one cooperative launch per step)",
            "d_lp_s_onebit": "onebit_decent_kernel<|N|> (one cooperative launch per step)",
            "codec": "encode_small_kernel + decode_small_kernel (register-resident; ring kernels above the capacity)",
            "onebit": "onebit_encode_kernel (fp64 |x| sum + sign bits) + onebit_decode_kernel"}[prim]


def ncu_traffic(prim: str, g: int):
    """DRAM bytes per launch measured by ncu (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(prim, {}).get(str(g))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                return
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def host_info() -> dict:
    """nproc, CPU model and RAM of the box the CPU legs run on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem_gb = None
    try:
        mem_gb = round(os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30, 1)
    except (ValueError, OSError):
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "ram_gib": mem_gb}


def cpu_reference_gbs(prim_id: int, g: int, n_sample: int, reps: int):
    """The unmodified reference (oracle/_ref) primitive through its SimCluster harness."""
    from oracle import Reference  # test/baseline infrastructure only
    r = Reference()
    secs = r.time_primitive(prim_id, g, n_sample, reps)
    return secs, r.backend()


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    g = world
    n_sample = min(args.n, args.ref_sample or args.n)
    prim_id, label = PRIMS[args.prim][1], PRIMS[args.prim][2]
    if args.prim in ("codec", "onebit"):
        g = 1
    secs, backend = cpu_reference_gbs(prim_id, g, n_sample, args.warmup + args.steps)
    timed = secs[args.warmup:] or secs
    t = statistics.median(timed)
    value = g * 4 * n_sample / t / 1e9
    full = n_sample == args.n
    workload = (f"C_LP_S ByteGrad MinMaxUInt8 allreduce of {args.n} fp32 gradients per GPU (VGG16-sized), g={world}"
                if args.prim == "c_lp_s" else f"{label} of {args.n} fp32 elements per GPU, g={world}")
    line = {
        "metric": f"effective gradient GB/s for {label}", "value": round(value, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+u8", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": workload if full else f"{label}, {n_sample} fp32 elements per worker (bounded "
                               f"sample of the {args.n}-element bucket), {g} worker threads on SimCluster",
                   "primitive": args.prim, "elements_per_gpu": n_sample, "parallelism": f"dp{world}",
                   "workers": g, "same_config_as_b200_arm": full},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": g, "kind": "reference",
                         "sample": f"{n_sample} elements x {g} workers (one thread per simulated GPU, the "
                                   f"reference's threading), median of {len(timed)} calls after {args.warmup} "
                                   f"warm-up, wall from spawn to join",
                         "backend": backend, **host_info()},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank: int, world: int):
    import torch
    import torch.distributed as dist
    import paper_2107_01499_b200 as b2

    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    g = world
    n = args.n
    prim = args.prim
    ep = b2.B200Endpoint(rank, world, dev, timeout_ms=120_000)
    codec = b2.Codec(b2.CodecKind.onebit if prim.endswith("_onebit") else b2.CodecKind.uniform8)
    stream = torch.cuda.current_stream()
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    b2._lib.check(b2.lib.b2_fill_synthetic(x.data_ptr(), n, 2026 + rank, 0, stream.cuda_stream))
    # C_* all-reduce SUMS in place: a buffer grows by g per call, so the timed
    # steps cycle through nbuf resident copies (each > L2, so no flush is
    # needed either) pre-scaled by an exact power of two so that no buffer
    # overflows over its uses (quantization is scale-equivariant: same codes).
    total_calls = args.warmup + args.steps + 2
    nbuf = 1 if prim.startswith("d_") or prim in ("codec", "onebit") else max(1, min(args.steps, 32))
    uses = -(-total_calls // nbuf) + 1
    shrink = 0 if nbuf == 1 else min(120, int(math.ceil(uses * math.log2(max(g, 2)))) + 1)
    x.mul_(2.0 ** -shrink)
    xs = [x] + [x.clone() for _ in range(nbuf - 1)]
    ring = b2.Topology(b2.TopologyKind.ring, g, 0)
    if prim in ("codec", "onebit"):  # one GPU, the standalone codec kernels
        codes = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
        hdr = torch.empty(4, dtype=torch.float32, device="cuda")
        launches_box = [0]

    def step(buf):
        if prim in ("c_lp_s", "c_lp_s_onebit"):
            b2.c_lp_s(ep, 0.0, buf, codec, None, blocking=False)
        elif prim == "c_fp_s":
            b2.c_fp_s(ep, 0.0, buf, blocking=False)
        elif prim == "d_fp_s":
            b2.d_fp_s(ep, 0.0, buf, ring, 0, b2.ReduceMode.average, blocking=False)
        elif prim in ("d_lp_s", "d_lp_s_onebit"):
            b2.d_lp_s(ep, 0.0, buf, ring, 0, codec, b2.ReduceMode.average, blocking=False)
        elif prim == "onebit":
            s_ = torch.cuda.current_stream().cuda_stream
            b2._lib.check(b2.lib.b2_onebit_encode(buf.data_ptr(), n, codes.data_ptr(), s_))
            b2._lib.check(b2.lib.b2_onebit_decode(codes.data_ptr(), n, buf.data_ptr(), s_))
            launches_box[0] += 2  # onebit_encode_kernel + onebit_decode_kernel
        else:
            s_ = torch.cuda.current_stream().cuda_stream
            b2._lib.check(b2.lib.b2_u8_encode(buf.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(), s_))
            b2._lib.check(b2.lib.b2_u8_decode(codes.data_ptr(), hdr.data_ptr(), n, buf.data_ptr(), s_))
            launches_box[0] += 2  # encode_ring_kernel (one cooperative launch) + decode_ring_kernel

    def n_launches():
        return launches_box[0] if prim in ("codec", "onebit") else ep.launches()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- device-resident timing (value)
    for i in range(args.warmup):
        step(xs[i % nbuf])
    ep.sync()
    # The standalone codec's step (encode + decode, two launches, ~15 us of
    # GPU work) is launch-bound from Python: its steps replay a CUDA graph of
    # the two launches (captured once; the same kernels, same buffers).
    # A graph holds GK consecutive steps (each a full encode + decode of the
    # bucket); the timed loop replays it steps / GK times, so the graph's own
    # launch (~6 us) is paid once per GK steps, as a training loop capturing
    # its steps would.
    graph = None
    eager_step = step
    GK = 1
    if prim in ("codec", "onebit") and not args.no_graph:
        GK = max(1, min(10, args.steps))
        while args.steps % GK:
            GK -= 1
        try:
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cap):  # per-stream scratch (onebit) is allocated before the capture
                step(xs[0])
            torch.cuda.synchronize()
            with torch.cuda.stream(cap):
                with torch.cuda.graph(graph, stream=cap):
                    for _ in range(GK):
                        step(xs[0])
            torch.cuda.current_stream().wait_stream(cap)
            launches_box[0] -= 2 * GK  # the capture launched nothing
            graph.replay()
            launches_box[0] += 2 * GK
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001  (capture unsupported: eager launches)
            print(json.dumps({"graph_capture": f"failed: {e}"}), file=sys.stderr)
            graph, GK = None, 1
    launches0 = n_launches()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.profile_range:  # ncu --profile-from-start off: only the timed steps
        torch.cuda.profiler.start()
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        if graph is not None:
            for _ in range(args.steps // GK):
                graph.replay()
                launches_box[0] += 2 * GK
        else:
            for i in range(args.steps):
                step(xs[i % nbuf])
        ev1.record(stream)
        ev1.synchronize()
    if args.profile_range:
        torch.cuda.profiler.stop()
    ep.sync()
    launches = n_launches() - launches0
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], device="cuda" if args.dist == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    barrier()

    # ---------------- end to end through the public API with host buffers
    # Every step hands the API a PINNED host bucket (the caller's gradients);
    # the library's host path (collectives._HostStaging) uploads it on its own
    # copy stream, runs the collective and downloads the result back into the
    # same host buffer on a second copy stream.  With blocking=False the
    # upload of step i+1 and the download of step i overlap the collective
    # (PCIe is full duplex), as a training loop issuing buckets would.  Two
    # host buckets alternate; each step's input is the result the buffer
    # received two steps before.
    NB = 2
    host = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(NB)]
    for h in host:
        h.copy_(xs[-1].cpu())

    def e2e_step(i):
        hb = host[i % NB]
        if prim in ("codec", "onebit"):  # the standalone codec has no host-bucket API: stage by hand
            xd = ep.__dict__.setdefault("_e2e_dev", torch.empty_like(x))
            xd.copy_(hb, non_blocking=True)
            eager_step(xd)
            hb.copy_(xd, non_blocking=True)
        else:
            step(hb)

    for i in range(max(2, args.warmup // 2)):
        e2e_step(i)
    ep.sync()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(2, args.steps if args.e2e_steps is None else min(args.steps, args.e2e_steps))
    e0.record(stream)
    for i in range(e_steps):
        e2e_step(i)
    ep.join(stream)  # the last downloads are part of the timed region
    e1.record(stream)
    e1.synchronize()
    ep.sync()
    ems = e0.elapsed_time(e1) / e_steps
    # the e2e leg's bound: one step's H2D and D2H on two streams at once, no
    # collective -- the full-duplex PCIe ceiling (tests/cpp/pcie_probe.py)
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    xd = [torch.empty_like(x) for _ in range(2)]
    barrier()
    pcie_ms = float("inf")
    for _ in range(3):  # best of 3: one 8 ms sample varies by +-10% with host load
        barrier()  # all ranks copy at once: they share the host's memory and root ports
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        h2d_s.wait_event(c0)
        d2h_s.wait_event(c0)
        with torch.cuda.stream(h2d_s):
            xd[0].copy_(host[0], non_blocking=True)
        with torch.cuda.stream(d2h_s):
            host[1].copy_(xd[1], non_blocking=True)
        for s_ in (h2d_s, d2h_s):
            ev = torch.cuda.Event()
            ev.record(s_)
            stream.wait_event(ev)
        c1.record(stream)
        c1.synchronize()
        pcie_ms = min(pcie_ms, c0.elapsed_time(c1))
    del xd
    if world > 1:
        t = torch.tensor([ems, pcie_ms], device="cuda" if args.dist == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems, pcie_ms = float(t[0].item()), float(t[1].item())

    trace = None
    if args.trace and prim not in ("codec", "onebit"):
        ep.enable_trace(True)
        barrier()
        for i in range(8):  # steady state: the last of 8 back-to-back calls is the one recorded
            step(xs[i % nbuf])
        trace = ep.read_trace()
        ep.enable_trace(False)
        if world > 1:
            allt = [None] * world
            dist.all_gather_object(allt, trace)
            trace = allt
        barrier()

    hbm_peak, peak_kind = measured_peaks()
    hbm_b, nvl_b = algorithmic_bytes(prim, n, g)
    t_s = ms / 1e3
    t_roof_hbm = hbm_b / (hbm_peak * 1e9)
    t_roof_nvl = nvl_b / (NVL_PEER_GBS * 1e9)
    if hbm_b == 0 and nvl_b == 0:
        roof = {"bound": "none", "achieved": 0.0, "peak": hbm_peak, "unit": "GB/s", "peak_kind": "n/a",
                "note": "no device work (C_FP_S with one worker returns x untouched, collectives.cpp:49); "
                        "the step time is the host call"}
    elif t_roof_nvl > t_roof_hbm:
        roof = {"bound": "nvlink", "achieved": round(nvl_b / t_s / 1e9, 2), "peak": NVL_PEER_GBS,
                "unit": "GB/s", "peak_kind": "measured peer copy (B200_PROFILING.md); nominal 900"}
    else:
        roof = {"bound": "hbm", "achieved": round(hbm_b / t_s / 1e9, 2), "peak": hbm_peak, "unit": "GB/s",
                "peak_kind": f"{peak_kind} HBM copy (MEASURED_PEAKS.json)"}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4) if roof["bound"] != "none" else None
    if nvl_b:  # the NVLink leg against both peaks (BASELINE.md 3 / SURVEY.md 8d quote the 900 GB/s nominal)
        roof["nvlink"] = {"achieved": round(nvl_b / t_s / 1e9, 2),
                          "frac_measured_770": round(nvl_b / t_s / 1e9 / NVL_PEER_GBS, 4),
                          "frac_nominal_900": round(nvl_b / t_s / 1e9 / NVL_NOMINAL_GBS, 4)}
        roof["hbm_leg"] = {"achieved": round(hbm_b / t_s / 1e9, 2), "frac": round(hbm_b / t_s / 1e9 / hbm_peak, 4)}
    roof["traffic"] = args.traffic if args.traffic is not None else ncu_traffic(prim, g)
    roof["algorithmic_bytes"] = {"hbm": hbm_b, "nvlink_ingress": nvl_b}
    roof["t_roof_us"] = round(max(t_roof_hbm, t_roof_nvl) * 1e6, 1)
    roof["kernel"] = kernel_label(prim, n, g)
    if prim == "c_lp_s" and g > 1:
        # the phase-serialized bound -- encode (HBM: x read +
        # codes written, 5N), scatter and gather (NVLink: N(g-1)/g each)
        ph = [5 * n / (hbm_peak * 1e9), n * (g - 1) / g / (NVL_PEER_GBS * 1e9), n * (g - 1) / g / (NVL_PEER_GBS * 1e9)]
        phn = ph[:1] + [t * NVL_PEER_GBS / NVL_NOMINAL_GBS for t in ph[1:]]
        roof["phase_serialized"] = {"phases_us": [round(t * 1e6, 1) for t in ph], "t_us": round(sum(ph) * 1e6, 1),
                                    "frac": round(sum(ph) / t_s, 4),
                                    "t_us_nominal_900": round(sum(phn) * 1e6, 1),
                                    "frac_nominal_900": round(sum(phn) / t_s, 4)}

    per_gpu = 4 * n / t_s / 1e9
    label = PRIMS[prim][2]
    line = {
        "metric": f"effective gradient GB/s for {label}", "value": round(g * per_gpu, 2), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32+u8",
        "data": (f"synthetic (splitmix64 uniform [-1,1) x 2^-{shrink}, seed 2026+rank; {nbuf} resident "
                 f"buffer(s) cycled, the sum grows by g per call)"),
        "config": {"workload": (f"C_LP_S ByteGrad MinMaxUInt8 allreduce of {n} fp32 gradients per GPU "
                                f"(VGG16-sized), g={g}" if prim == "c_lp_s" else f"{label} of {n} fp32 elements "
                                f"per GPU, g={g}"), "primitive": prim, "elements_per_gpu": n, "parallelism": f"dp{g}",
                   "per_gpu_gbs": round(per_gpu, 2), "l2": f"inputs {4 * n / 1e6:.0f} MB/GPU per step, {nbuf} buffer(s) cycled; > 126 MB L2, no flush"},
        "roofline": roof,
        "e2e": {"value": round(g * 4 * n / (ems / 1e3) / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": 4 * n, "ms_per_step": round(ems, 3), "steps": e_steps,
                "bound": "pcie (concurrent pinned H2D + D2H of one step's bytes, measured in this run)",
                "path": ("b2.c_lp_s / c_fp_s / d_*(ep, 0.0, pinned_host_bucket, ..., blocking=False): the library's "
                         "own host staging (cached device ring, copy streams), ep.sync() after the last step"
                         if prim not in ("codec", "onebit") else "hand-staged: the standalone codec has no host API"),
                "ceiling": round(g * 4 * n / (pcie_ms / 1e3) / 1e9, 2), "frac": round(pcie_ms / ems, 3)},
        "gpu_launches": int(launches),
        "cuda_graph_steps": GK if graph is not None else 0,
        "clocks": clk.summary(),
    }
    if world > 1:  # every rank's GPU clocks during its timed region (run-to-run spread)
        per = [None] * world
        dist.all_gather_object(per, {"rank": rank, "device": dev, **clk.summary()})
        line["clocks_per_rank"] = per
    if rank == 0 and world == 1 and not args.no_cpu_baseline and prim != "c_fp_s":
        n_sample = min(n, args.cpu_sample or n)
        secs, backend = cpu_reference_gbs(PRIMS[prim][1], 1, n_sample, 4)
        tc = statistics.median(secs[1:])  # 1 warm-up, median of 3
        line["cpu_baseline"] = {"value": round(4 * n_sample / tc / 1e9, 4), "unit": "GB/s", "cores": 1,
                                "kind": "reference",
                                "sample": f"{label} g=1 over {n_sample} elements (the full bucket), 1 warm-up "
                                          f"then median of 3 calls (reference SimCluster harness)",
                                "backend": backend, **host_info()}
    if rank == 0:
        print(json.dumps(line), flush=True)
        if trace is not None:
            print(json.dumps({"phase_trace_us(median,max)": trace}), file=sys.stderr, flush=True)
    ep.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--prim", default="c_lp_s", choices=sorted(PRIMS))
    ap.add_argument("--n", "--elements", dest="n", type=int, default=None,
                    help="elements per GPU (default: the BASELINE config size); use --elements under torchrun")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="steps in the e2e leg (default: --steps; the pipeline fill is amortised over them)")
    ap.add_argument("--cpu-sample", type=int, default=None, help="elements (default: the full bucket)")
    ap.add_argument("--ref-sample", type=int, default=None, help="elements per worker (default: the full bucket)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace", action="store_true", help="print per-phase device timestamps (stderr)")
    ap.add_argument("--no-graph", action="store_true", help="codec prims: eager launches instead of a CUDA graph")
    ap.add_argument("--profile-range", action="store_true",
                    help="cudaProfilerStart/Stop around the timed steps (ncu --profile-from-start off)")
    ap.add_argument("--dist", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend of the plumbing (barriers, max over ranks)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes/launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.n is None:
        args.n = PRIMS[args.prim][0]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "b200" and args.dist == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
            dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank))))
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
