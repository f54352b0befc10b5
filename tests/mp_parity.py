"""Multi-GPU parity driver: one process per GPU (torchrun), every primitive
against the CPU oracle on identical, deterministically generated inputs.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \
        --master-port 29511 tests/mp_parity.py [--quick] [--large]

Each rank regenerates every rank's input from the shared seeds (synthetic
splitmix64 generator, identical on host and device), computes the oracle
result for ITSELF and compares bit for bit.  For large buckets each rank
checks its own partition with the partition-local restatement
and all ranks compare digests of their full outputs (every rank must hold the
identical bucket after C_*).  Rank 0 prints one JSON line; exit code 1 on
any mismatch.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
import traceback

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2107_01499_b200 as b2  # noqa: E402
from oracle import Oracle  # noqa: E402  (test infrastructure: the checker)

U8 = b2.Codec(b2.CodecKind.uniform8)
ID = b2.Codec(b2.CodecKind.identity)
OB = b2.Codec(b2.CodecKind.onebit)


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


class Checker:
    def __init__(self, rank):
        self.rank = rank
        self.fail: list[str] = []
        self.passed = 0

    def eq(self, name, got, want):
        if np.array_equal(bits(got), bits(want)):
            self.passed += 1
        else:
            bad = np.flatnonzero(bits(got) != bits(want))
            self.fail.append(f"rank{self.rank} {name}: {bad.size} mismatches, first at {bad[:5].tolist()} "
                             f"got {np.asarray(got).ravel()[bad[:3]].tolist()} "
                             f"want {np.asarray(want).ravel()[bad[:3]].tolist()}")

    def close(self, name, got, want, ulps=4):
        """Onebit scales come from fp64 |y| sums whose order differs from the
        reference's (codec.cpp:82-83); inexact sums may round one float apart.
        Bound: ulps x spacing(max |want|).  Exact matches are counted."""
        got, want = np.asarray(got, np.float32), np.asarray(want, np.float32)
        if np.array_equal(bits(got), bits(want)):
            self.passed += 1
            self.exact = getattr(self, "exact", 0) + 1
            return
        tol = ulps * float(np.spacing(np.float32(np.abs(want).max(initial=1.0))))
        err = float(np.abs(got.astype(np.float64) - want).max(initial=0.0))
        if err <= tol:
            self.passed += 1
        else:
            self.fail.append(f"rank{self.rank} {name}: max err {err} > {tol}")


def replicas_identical(ck, name, t, g, rank):
    """Every rank must hold the identical bucket after a C_* primitive."""
    digest = hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()
    allv = [None] * g
    dist.all_gather_object(allv, digest)
    if len(set(allv)) != 1:
        ck.fail.append(f"rank{rank} {name}: replicas differ {allv}")
    else:
        ck.passed += 1


def run_large(ep, ck, orc, rank, g):
    """BASELINE.json's configs at their full sizes, every rank checked against
    the oracle.  C_*: the owner checks its own partition against the
    partition-local restatement and all ranks compare digests
    of their whole outputs (so every replica of every partition is checked);
    where the whole problem fits (25M) the full oracle runs instead.  D_*:
    the per-rank restatement over the rank's neighbours' inputs.  Inputs are
    splitmix64 synthetic gradients generated identically on the device and
    on the host (orc_synth == b2_fill_synthetic)."""
    stream = torch.cuda.current_stream().cuda_stream

    def fill(n, seed):
        t = torch.empty(n, device="cuda")
        b2._lib.check(b2.lib.b2_fill_synthetic(t.data_ptr(), n, seed, 0, stream))
        return t

    bucket = 5000
    # -- config 2: C_FP_S, 25M fp32, full oracle (fp64 ascending rank fold)
    n = 25_000_000
    xs = [orc.synth(n, 2026 + r) for r in range(g)]
    want = [x.copy() for x in xs]
    orc.c_fp_s(want)
    for it in range(2):
        t = torch.as_tensor(xs[rank]).cuda()
        b2.c_fp_s(ep, 0.0, t, bucket=bucket)
        ck.eq(f"large c_fp_s n={n} it={it}", t.cpu().numpy(), want[rank])
    del want
    # -- config 4: D_FP_S ring averaging, 25M, two chained rounds
    topo = b2.Topology(b2.TopologyKind.ring, g, 0)
    nb = topo.neighbors(rank, 0)
    t = torch.as_tensor(xs[rank]).cuda()
    cur = xs
    for rnd in range(2):
        b2.d_fp_s(ep, 0.0, t, topo, rnd, b2.ReduceMode.average, bucket=bucket + 1)
        cur = [orc.d_fp_s_rank([cur[j] for j in topo.neighbors(r, rnd)], 1) for r in range(g)]
        ck.eq(f"large d_fp_s ring n={n} round={rnd}", t.cpu().numpy(), cur[rank])
    del cur, xs

    # -- config 3: C_LP_S 100M uint8 (stateless, two calls), onebit, uint8 + error feedback
    n = 100_000_000
    lo, sz = b2.partition_range(n, g, rank)
    for it in range(2):
        seed0 = 2026 + 100 * it
        t = fill(n, seed0 + rank)
        b2.c_lp_s(ep, 0.0, t, U8, None, bucket=bucket + 2)
        acc = np.zeros(sz, np.float64)
        for r in range(g):  # partition-local restatement: D(Q2((float) sum_j D(Q1(x_j|k))))
            l1, h1, c1 = orc.encode(orc.synth(sz, seed0 + r, lo))
            acc += orc.decode(l1, h1, c1).astype(np.float64)
        l2, h2, c2 = orc.encode(acc.astype(np.float32))
        ck.eq(f"large c_lp_s u8 n={n} it={it} own partition", t[lo:lo + sz].cpu().numpy(), orc.decode(l2, h2, c2))
        replicas_identical(ck, f"large c_lp_s u8 n={n} it={it}", t, g, rank)
    t = fill(n, 2026 + rank)
    b2.c_lp_s(ep, 0.0, t, OB, None, bucket=bucket + 3)
    acc = np.zeros(sz, np.float64)
    for r in range(g):
        p = orc.synth(sz, 2026 + r, lo)
        acc += orc.onebit_decode_wire(orc.onebit_encode_wire(p), sz).astype(np.float64)
    s = acc.astype(np.float32)
    ck.close(f"large c_lp_s onebit n={n} own partition", t[lo:lo + sz].cpu().numpy(),
             orc.onebit_decode_wire(orc.onebit_encode_wire(s), sz))
    replicas_identical(ck, f"large c_lp_s onebit n={n}", t, g, rank)
    del acc, s
    # uint8 + ErrorState over 3 rounds (acceptance c4 semantics, collectives.cpp:109-151):
    # my whole delta, my epsilon and my own partition of x' are checked
    es = b2.ErrorState(n, sz)
    parts = [(b2.partition_range(n, g, k)) for k in range(g)]
    my_delta = np.zeros(n, np.float32)               # delta of this rank, whole bucket
    d_mine = [np.zeros(sz, np.float32) for _ in range(g)]  # delta_j over MY partition, every j
    eps = np.zeros(sz, np.float32)
    for rnd in range(3):
        seed0 = 4040 + 100 * rnd
        t = fill(n, seed0 + rank)
        b2.c_lp_s(ep, 0.0, t, U8, es, bucket=bucket + 4)
        for k, (lk, nk) in enumerate(parts):  # my delta: chunk by chunk, codec.cpp:125-137
            orc.compensate_encode(orc.synth(nk, seed0 + rank, lk), my_delta[lk:lk + nk])
        acc = np.zeros(sz, np.float64)
        for r in range(g):
            _, _, _, dec = orc.compensate_encode(orc.synth(sz, seed0 + r, lo), d_mine[r])
            acc += dec[:sz].astype(np.float64)
        _, _, _, d2 = orc.compensate_encode(acc.astype(np.float32), eps)
        ck.eq(f"large c_lp_s u8+EC n={n} round={rnd} own partition", t[lo:lo + sz].cpu().numpy(), d2[:sz])
        ck.eq(f"large c_lp_s u8+EC n={n} round={rnd} delta", es.delta.cpu().numpy(), my_delta)
        ck.eq(f"large c_lp_s u8+EC n={n} round={rnd} epsilon", es.epsilon.cpu().numpy(), eps)
        replicas_identical(ck, f"large c_lp_s u8+EC n={n} round={rnd}", t, g, rank)
    del es, my_delta, d_mine, eps, acc, t
    torch.cuda.empty_cache()

    # -- config 5: D_LP_S ring averaging, bucket sweep 1M .. 340M (per-rank restatement)
    for i, n in enumerate((1_000_000, 25_000_000, 100_000_000, 340_000_000)):
        t = fill(n, 6060 + rank)
        b2.d_lp_s(ep, 0.0, t, topo, 0, U8, b2.ReduceMode.average, bucket=bucket + 10 + i)
        want = orc.d_lp_s_rank([orc.synth(n, 6060 + j) for j in nb], 1, 1)
        ck.eq(f"large d_lp_s ring n={n}", t.cpu().numpy(), want)
        del t, want
        ep.release_bucket(bucket + 10 + i)
        torch.cuda.empty_cache()


def run(args):
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    orc = Oracle()
    ep = b2.B200Endpoint(rank, world, dev, timeout_ms=120_000)
    ck = Checker(rank)
    g = world

    if args.large:
        run_large(ep, ck, orc, rank, g)
        return ck, ep.launches()

    sizes = [1, 3, 5, 37, 1000, 4097, 65536 + 7, 1_000_003]
    if not args.quick:
        sizes += [4_000_000, 25_000_000]
    bucket = 0
    for n in sizes:
        bucket += 1
        xs = [orc.synth(n, 2026 + r) for r in range(g)]
        # ---- C_LP_S uint8 (stateless), repeated calls on one bucket (epoch protocol)
        for it in range(3):
            xs_it = [orc.synth(n, 7000 + 31 * it + r) for r in range(g)]
            want = [x.copy() for x in xs_it]
            orc.c_lp_s(want, codec=1)
            t = torch.as_tensor(xs_it[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, U8, None, bucket=bucket)
            ck.eq(f"c_lp_s u8 n={n} it={it}", t.cpu().numpy(), want[rank])
        # ---- C_LP_S identity == C_FP_S fp64 ordered sum
        want = [x.copy() for x in xs]
        orc.c_lp_s(want, codec=0)
        t = torch.as_tensor(xs[rank]).cuda()
        b2.c_lp_s(ep, 0.0, t, ID, None, bucket=bucket)
        ck.eq(f"c_lp_s identity n={n}", t.cpu().numpy(), want[rank])
        want = [x.copy() for x in xs]
        orc.c_fp_s(want)
        for it in range(2):
            t = torch.as_tensor(xs[rank]).cuda()
            b2.c_fp_s(ep, 0.0, t, bucket=bucket)
            ck.eq(f"c_fp_s n={n} it={it}", t.cpu().numpy(), want[rank])
        # ---- D_FP_S / D_LP_S over ring, full, random
        for kind in (b2.TopologyKind.ring, b2.TopologyKind.full, b2.TopologyKind.random):
            topo = b2.Topology(kind, g, 123)
            for rnd in range(3):
                nb = topo.neighbors(rank, rnd)
                for mode in (b2.ReduceMode.average, b2.ReduceMode.sum):
                    t = torch.as_tensor(xs[rank]).cuda()
                    b2.d_fp_s(ep, 0.0, t, topo, rnd, mode, bucket=bucket)
                    ck.eq(f"d_fp_s {kind.name} r{rnd} {mode.name} n={n}", t.cpu().numpy(),
                          orc.d_fp_s_rank([xs[j] for j in nb], int(mode)))
                    t = torch.as_tensor(xs[rank]).cuda()
                    b2.d_lp_s(ep, 0.0, t, topo, rnd, U8, mode, bucket=bucket)
                    ck.eq(f"d_lp_s {kind.name} r{rnd} {mode.name} n={n}", t.cpu().numpy(),
                          orc.d_lp_s_rank([xs[j] for j in nb], 1, int(mode)))
        t = torch.as_tensor(xs[rank]).cuda()
        topo = b2.Topology(b2.TopologyKind.ring, g, 0)
        b2.d_lp_s(ep, 0.0, t, topo, 0, ID, b2.ReduceMode.average, bucket=bucket)
        ck.eq(f"d_lp_s identity n={n}", t.cpu().numpy(),
              orc.d_fp_s_rank([xs[j] for j in topo.neighbors(rank, 0)], 1))

    # ---- stochastic rounding inside C_LP_S / D_LP_S (codec.cpp:67-78): the
    # expectation over calls is the exact sum / neighbourhood mean; every rank
    # of a C_LP_S call holds the same bucket
    import random
    ST = b2.Codec(b2.CodecKind.uniform8, b2.Rounding.stochastic)
    n, calls = 20_000, 60
    bucket += 1
    xs = [orc.synth(n, 8300 + r) for r in range(g)]
    rng = random.Random(100 + rank)  # per-rank generators (the seed mixes the rank anyway)
    acc = np.zeros(n, np.float64)
    accd = np.zeros(n, np.float64)
    ring = b2.Topology(b2.TopologyKind.ring, g, 0)
    nb = ring.neighbors(rank, 0)
    for c in range(calls):
        t = torch.as_tensor(xs[rank]).cuda()
        b2.c_lp_s(ep, 0.0, t, ST, None, rng, bucket=bucket)
        out = t.cpu().numpy()
        acc += out
        if c == 0:
            replicas_identical(ck, "c_lp_s stochastic", t, g, rank)
        t = torch.as_tensor(xs[rank]).cuda()
        b2.d_lp_s(ep, 0.0, t, ring, 0, ST, b2.ReduceMode.average, rng, bucket=bucket + 1)
        accd += t.cpu().numpy()
    bucket += 1
    want = np.sum([x.astype(np.float64) for x in xs], axis=0)
    wantd = np.mean([xs[j].astype(np.float64) for j in nb], axis=0)
    # per element the two stochastic roundings add variance <= (g step1^2 + step2^2) / 4
    step1 = 2.0 / 255.0
    step2 = 2.0 * g / 255.0
    tol = 6.0 * np.sqrt((g * step1 ** 2 + step2 ** 2) / 4.0 / calls)
    if np.abs(acc / calls - want).mean() < tol / 3 and np.abs(accd / calls - wantd).mean() < tol / 3:
        ck.passed += 1
    else:
        ck.fail.append(f"rank{rank} stochastic C_LP_S/D_LP_S biased: {np.abs(acc / calls - want).mean()} "
                       f"{np.abs(accd / calls - wantd).mean()} tol {tol / 3}")

    # ---- D_* between the register capacity and the ring cut-over: the
    # streaming per-CTA kernel (small_coll.cu decent_stream_kernel)
    for n in (6_000_001, 16_000_000):
        bucket += 1
        xs = [orc.synth(n, 8100 + r) for r in range(g)]
        for kind in (b2.TopologyKind.ring, b2.TopologyKind.random):
            topo = b2.Topology(kind, g, 11)
            for rnd in range(2):
                nb = topo.neighbors(rank, rnd)
                t = torch.as_tensor(xs[rank]).cuda()
                b2.d_lp_s(ep, 0.0, t, topo, rnd, U8, b2.ReduceMode.average, bucket=bucket)
                ck.eq(f"d_lp_s stream {kind.name} r{rnd} n={n}", t.cpu().numpy(),
                      orc.d_lp_s_rank([xs[j] for j in nb], 1, 1))
                t = torch.as_tensor(xs[rank]).cuda()
                b2.d_fp_s(ep, 0.0, t, topo, rnd, b2.ReduceMode.sum, bucket=bucket)
                ck.eq(f"d_fp_s stream {kind.name} r{rnd} n={n}", t.cpu().numpy(),
                      orc.d_fp_s_rank([xs[j] for j in nb], 0))

    # ---- chunk-aligned shapes (n % 16g == 0): the staggered C_LP_S kernel
    # (central_stag.cu), stateless and with error feedback, repeated calls
    for n in (16 * g, 16 * g * 37, 16 * g * 4099, 16 * g * 65537):
        bucket += 1
        for it in range(3):
            xs_it = [orc.synth(n, 7300 + 31 * it + r) for r in range(g)]
            want = [x.copy() for x in xs_it]
            orc.c_lp_s(want, codec=1)
            t = torch.as_tensor(xs_it[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, U8, None, bucket=bucket)
            ck.eq(f"c_lp_s u8 aligned n={n} it={it}", t.cpu().numpy(), want[rank])
        bucket += 1
        own = b2.owned_partition_len(n, g, rank)
        es = b2.ErrorState(n, own)
        deltas = [np.zeros(n, np.float32) for _ in range(g)]
        eps = [np.zeros(b2.owned_partition_len(n, g, r), np.float32) for r in range(g)]
        for t_ in range(4):
            grads = [orc.synth(n, 7400 + 1000 * r + t_) for r in range(g)]
            want = [x.copy() for x in grads]
            orc.c_lp_s(want, codec=1, deltas=deltas, eps=eps)
            t = torch.as_tensor(grads[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, U8, es, bucket=bucket, blocking=False)
            ck.eq(f"c_lp_s+EC aligned n={n} round={t_} x", t.cpu().numpy(), want[rank])
        ck.eq(f"c_lp_s+EC aligned n={n} delta", es.delta.cpu().numpy(), deltas[rank])
        ck.eq(f"c_lp_s+EC aligned n={n} eps", es.epsilon.cpu().numpy(), eps[rank])

    # ---- one window switching between the register-resident C_* kernel
    # (small_central.cu) and the TMA ring as the SM budget changes: separate
    # call counters per protocol, buffers reused across the two
    n = 1_000_003
    bucket += 1
    own = b2.owned_partition_len(n, g, rank)
    es = b2.ErrorState(n, own)
    deltas = [np.zeros(n, np.float32) for _ in range(g)]
    eps = [np.zeros(b2.owned_partition_len(n, g, r), np.float32) for r in range(g)]
    for t_, sms in enumerate((0, 4, 4, 0, 0, 4, 0)):
        ep.set_sm_budget(sms)
        grads = [orc.synth(n, 7600 + 1000 * r + t_) for r in range(g)]
        want = [x.copy() for x in grads]
        orc.c_lp_s(want, codec=1, deltas=deltas, eps=eps)
        t = torch.as_tensor(grads[rank]).cuda()
        b2.c_lp_s(ep, 0.0, t, U8, es, bucket=bucket)
        ck.eq(f"c_lp_s+EC budget-switch n={n} round={t_} sms={sms}", t.cpu().numpy(), want[rank])
        want = [x.copy() for x in grads]
        orc.c_fp_s(want)
        t = torch.as_tensor(grads[rank]).cuda()
        b2.c_fp_s(ep, 0.0, t, bucket=bucket + 1)
        ck.eq(f"c_fp_s budget-switch n={n} round={t_} sms={sms}", t.cpu().numpy(), want[rank])
    ep.set_sm_budget(0)
    ck.eq(f"c_lp_s+EC budget-switch n={n} delta", es.delta.cpu().numpy(), deltas[rank])
    ck.eq(f"c_lp_s+EC budget-switch n={n} eps", es.epsilon.cpu().numpy(), eps[rank])
    bucket += 1

    # ---- C_LP_S uint8 + error feedback, acceptance c4 style (many rounds, state carried)
    for n, rounds in ((37, 200), (100_003, 10)):
        bucket += 1
        own = b2.owned_partition_len(n, g, rank)
        es = b2.ErrorState(n, own)
        deltas = [np.zeros(n, np.float32) for _ in range(g)]
        eps = [np.zeros(b2.owned_partition_len(n, g, r), np.float32) for r in range(g)]
        for t_ in range(rounds):
            grads = [orc.synth(n, 7000 + 1000 * r + t_) for r in range(g)]
            want = [x.copy() for x in grads]
            orc.c_lp_s(want, codec=1, deltas=deltas, eps=eps)
            t = torch.as_tensor(grads[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, U8, es, bucket=bucket)
            ck.eq(f"c_lp_s+EC n={n} round={t_} x", t.cpu().numpy(), want[rank])
            ck.eq(f"c_lp_s+EC n={n} round={t_} delta", es.delta.cpu().numpy(), deltas[rank])
            ck.eq(f"c_lp_s+EC n={n} round={t_} eps", es.epsilon.cpu().numpy(), eps[rank])

    # ---- C_LP_S onebit (the 1-bit Adam aggregation, algorithms.cpp:141-148)
    ob_sizes = [1, 3, 5, 37, 1000, 4097, 65536 + 7, 1_000_003] + ([] if args.quick else [4_000_000])
    for n in ob_sizes:
        bucket += 1
        for it in range(2):
            xs_it = [orc.synth(n, 9100 + 31 * it + r) for r in range(g)]
            want = [x.copy() for x in xs_it]
            orc.c_lp_s(want, codec=2)
            t = torch.as_tensor(xs_it[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, OB, None, bucket=bucket)
            ck.close(f"c_lp_s onebit n={n} it={it}", t.cpu().numpy(), want[rank])
    for n, rounds in ((37, 20), (100_003, 5)):
        bucket += 1
        own = b2.owned_partition_len(n, g, rank)
        es = b2.ErrorState(n, own)
        deltas = [np.zeros(n, np.float32) for _ in range(g)]
        eps = [np.zeros(b2.owned_partition_len(n, g, r), np.float32) for r in range(g)]
        for t_ in range(rounds):
            grads = [orc.synth(n, 9500 + 1000 * r + t_) for r in range(g)]
            want = [x.copy() for x in grads]
            orc.c_lp_s(want, codec=2, deltas=deltas, eps=eps)
            t = torch.as_tensor(grads[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, OB, es, bucket=bucket, blocking=False)
            ck.close(f"c_lp_s onebit+EC n={n} round={t_} x", t.cpu().numpy(), want[rank])
            ck.close(f"c_lp_s onebit+EC n={n} round={t_} delta", es.delta.cpu().numpy(), deltas[rank])
            ck.close(f"c_lp_s onebit+EC n={n} round={t_} eps", es.epsilon.cpu().numpy(), eps[rank])
    # back-to-back non-blocking onebit calls on one bucket, one sync at the end
    bucket += 1
    n = 200_003
    ts = [torch.as_tensor(orc.synth(n, 60 + r)).cuda() for r in range(2)]
    for i in range(6):
        b2.c_lp_s(ep, 0.0, ts[i % 2], OB, None, bucket=bucket, blocking=False)
    ep.sync()
    for r in range(2):  # each buffer went through 3 calls; every rank starts from the same x
        w = [orc.synth(n, 60 + r) for _ in range(g)]
        for _ in range(3):
            orc.c_lp_s(w, codec=2)
        ck.close(f"c_lp_s onebit back-to-back buf{r}", ts[r].cpu().numpy(), w[rank])

    # ---- D_LP_S onebit over ring / full / random, both modes, repeated rounds
    for n in [1, 5, 37, 1000, 4097, 65536 + 7, 1_000_003] + ([] if args.quick else [4_000_000]):
        bucket += 1
        xs = [orc.synth(n, 8800 + r) for r in range(g)]
        for kind in (b2.TopologyKind.ring, b2.TopologyKind.full, b2.TopologyKind.random):
            topo = b2.Topology(kind, g, 77)
            for rnd in range(3):
                nb = topo.neighbors(rank, rnd)
                for mode in (b2.ReduceMode.average, b2.ReduceMode.sum):
                    t = torch.as_tensor(xs[rank]).cuda()
                    b2.d_lp_s(ep, 0.0, t, topo, rnd, OB, mode, bucket=bucket)
                    ck.close(f"d_lp_s onebit {kind.name} r{rnd} {mode.name} n={n}", t.cpu().numpy(),
                             orc.d_lp_s_rank([xs[j] for j in nb], 2, int(mode)))
    # back-to-back non-blocking onebit D_LP_S with a changing (random) topology, state carried
    bucket += 1
    n = 300_007
    topo = b2.Topology(b2.TopologyKind.random, g, 5)
    cur = [orc.synth(n, 610 + r) for r in range(g)]
    t = torch.as_tensor(cur[rank]).cuda()
    for rnd in range(12):
        b2.d_lp_s(ep, 0.0, t, topo, rnd, OB, b2.ReduceMode.average, bucket=bucket, blocking=False)
        cur = [orc.d_lp_s_rank([cur[j] for j in topo.neighbors(r, rnd)], 2, 1) for r in range(g)]
    ep.sync()
    ck.close("d_lp_s onebit back-to-back random topology", t.cpu().numpy(), cur[rank])

    # ---- hierarchical_c over virtual node layouts (collectives.cpp:290-385),
    # on grid inputs (exact fp64 sums) and on mixed-magnitude gaussians
    # (inexact sums: the lossless multi-node branch folds in a different fp64
    # order than the reference, declared tolerance 1 fp32 ulp; lossy branches
    # bit-exact, -0.0 included -- the down phase is a byte broadcast)
    layouts = {2: [[0, 1], [0, 0]], 3: [[0, 0, 1], [0, 1, 2]], 4: [[0, 0, 1, 1], [0, 1, 1, 2], [1, 0, 1, 0]]}

    def gauss(n, seed):
        rs = np.random.default_rng(seed)
        v = (rs.standard_normal(n) * 10.0 ** rs.uniform(-6, 6, n)).astype(np.float32)
        v[::97] = -0.0
        return v

    for nodes in layouts.get(g, [[0] * g]):
        multi = len(set(nodes)) > 1
        for codec_kind, codec in ((0, ID), (1, U8), (2, OB)):
            for n, gen in ((37, "grid"), (100_003, "grid"), (100_003, "gauss")):
                bucket += 1
                xs = [orc.synth(n, 7700 + r) if gen == "grid" else gauss(n, 7800 + r) for r in range(g)]
                want = [x.copy() for x in xs]
                orc.hierarchical_c(want, nodes, codec_kind)
                t = torch.as_tensor(xs[rank]).cuda()
                b2.hierarchical_c(ep, 0.0, t, codec, None, bucket=bucket, nodes=nodes)
                got = t.cpu().numpy()
                name = f"hierarchical_c nodes={nodes} codec={codec_kind} n={n} {gen}"
                if codec_kind == 2:
                    ck.close(name, got, want[rank])
                elif codec_kind == 0 and multi and gen == "gauss":
                    w = want[rank]
                    ok = np.all(np.abs(got.astype(np.float64) - w) <= np.spacing(np.abs(w)))
                    if ok:
                        ck.passed += 1
                    else:
                        ck.fail.append(f"rank{rank} {name}: beyond 1 ulp")
                else:
                    ck.eq(name, got, want[rank])

    # ---- interleaved buckets, non-blocking issue, one sync (overlap of buckets)
    bucket += 1
    n = 300_001
    xs = [[orc.synth(n, 50 + 10 * b + r) for r in range(g)] for b in range(3)]
    ts = [torch.as_tensor(xs[b][rank]).cuda() for b in range(3)]
    for b in range(3):
        b2.c_lp_s(ep, 0.0, ts[b], U8, None, bucket=bucket + b, blocking=False)
    ep.sync()
    for b in range(3):
        want = [x.copy() for x in xs[b]]
        orc.c_lp_s(want, codec=1)
        ck.eq(f"interleaved bucket {b}", ts[b].cpu().numpy(), want[rank])

    # ---- back-to-back stress: many non-blocking calls on one bucket, two
    # alternating buffers, one sync at the end (epoch counters, region
    # counters, per-parity D_* buffers and counters with a random topology
    # whose |N| changes every round, a neighbour running a call ahead)
    for n, prim in ((100_003, "c_lp_s"), (100_003, "c_fp_s"), (100_003, "d_lp_s"), (100_003, "d_fp_s"),
                    (1_000_037, "c_lp_s"), (1_000_037, "d_lp_s"), (16 * g * 65537, "c_lp_s")):
        bucket += 1
        calls = 16
        host = [[orc.synth(n, 900 + 10 * b + r) for r in range(g)] for b in range(2)]
        ts = [torch.as_tensor(host[b][rank]).cuda() for b in range(2)]
        topo = b2.Topology(b2.TopologyKind.random, g, 99)
        for i in range(calls):
            b = i % 2
            if prim == "c_lp_s":
                b2.c_lp_s(ep, 0.0, ts[b], U8, None, bucket=bucket, blocking=False)
                want = [x.copy() for x in host[b]]
                orc.c_lp_s(want, codec=1)
            elif prim == "c_fp_s":
                b2.c_fp_s(ep, 0.0, ts[b], bucket=bucket, blocking=False)
                want = [x.copy() for x in host[b]]
                orc.c_fp_s(want)
            else:
                fn = b2.d_lp_s if prim == "d_lp_s" else b2.d_fp_s
                if prim == "d_lp_s":
                    fn(ep, 0.0, ts[b], topo, i, U8, b2.ReduceMode.average, bucket=bucket, blocking=False)
                else:
                    fn(ep, 0.0, ts[b], topo, i, b2.ReduceMode.average, bucket=bucket, blocking=False)
                want = []
                for r in range(g):
                    nb = topo.neighbors(r, i)
                    srcs = [host[b][j] for j in nb]
                    want.append(orc.d_lp_s_rank(srcs, 1, 1) if prim == "d_lp_s" else orc.d_fp_s_rank(srcs, 1))
            host[b] = want
        ep.sync()
        for b in range(2):
            ck.eq(f"stress {prim} buffer {b} after {calls} back-to-back calls", ts[b].cpu().numpy(), host[b][rank])

    # ---- back-to-back with error feedback (uint8 and identity codec), state carried
    for codec_kind, codec in ((1, U8), (0, ID)):
        n = 70_001
        bucket += 1
        own = b2.owned_partition_len(n, g, rank)
        es = b2.ErrorState(n, own)
        deltas = [np.zeros(n, np.float32) for _ in range(g)]
        eps = [np.zeros(b2.owned_partition_len(n, g, r), np.float32) for r in range(g)]
        outs = []
        for t_ in range(12):
            grads = [orc.synth(n, 5000 + 100 * r + t_) for r in range(g)]
            want = [x.copy() for x in grads]
            orc.c_lp_s(want, codec=codec_kind, deltas=deltas, eps=eps)
            t = torch.as_tensor(grads[rank]).cuda()
            b2.c_lp_s(ep, 0.0, t, codec, es, bucket=bucket, blocking=False)
            outs.append((t, want[rank]))
        ep.sync()
        for t_, (t, w) in enumerate(outs):
            ck.eq(f"stress c_lp_s+EC codec={codec_kind} round={t_} x", t.cpu().numpy(), w)
        ck.eq(f"stress c_lp_s+EC codec={codec_kind} delta", es.delta.cpu().numpy(), deltas[rank])
        ck.eq(f"stress c_lp_s+EC codec={codec_kind} eps", es.epsilon.cpu().numpy(), eps[rank])

    # ---- engine: bucketed C_LP_S overlapping a synthetic backward on the
    # compute stream (comm on its own stream); every bucket == the oracle's
    # c_lp_s over that bucket's arena of every rank
    from paper_2107_01499_b200.engine import OverlapEngine
    sizes = [3000, 17, 70_001, 5, 250_000, 1024, 33_333]
    eng = OverlapEngine(ep, sizes, capacity_bytes=4 * 100_000)
    host = {}
    for it in range(2):
        for layer in reversed(range(len(sizes))):
            vals = orc.synth(sizes[layer], 31_000 + 100 * it + 10 * layer + rank)
            host[layer] = vals
            torch.cuda._sleep(20_000)  # "backward" of this layer on the compute stream
            eng.grad(layer).copy_(torch.as_tensor(vals), non_blocking=False)
            eng.layer_done(layer)
        eng.finish()
        torch.cuda.synchronize()
        for b in eng.buckets:
            xs_b = []
            for r in range(g):
                parts = [orc.synth(sizes[layer], 31_000 + 100 * it + 10 * layer + r) for layer in b.layers]
                xs_b.append(np.concatenate(parts).astype(np.float32))
            orc.c_lp_s(xs_b, codec=1)
            ck.eq(f"engine it={it} bucket {b.id} layers {b.layers}", eng.arenas[b.id].cpu().numpy(), xs_b[rank])

    return ck, ep.launches()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--large", action="store_true",
                    help="only BASELINE.json's configs at full size (25M C_FP_S / D_FP_S, 100M C_LP_S "
                         "uint8 / onebit / EC, D_LP_S 1M-340M)")
    args = ap.parse_args()
    dist.init_process_group("gloo")
    t0 = time.time()
    try:
        ck, launches = run(args)
        fails, passed, exact = ck.fail, ck.passed, getattr(ck, "exact", 0)
    except Exception:
        fails, passed, launches, exact = [f"rank{dist.get_rank()} exception: {traceback.format_exc()}"], 0, 0, 0
    allres = [None] * dist.get_world_size()
    dist.all_gather_object(allres, (passed, fails, launches, exact))
    if dist.get_rank() == 0:
        total_pass = sum(p for p, _, _, _ in allres)
        all_fail = [f for _, fs, _, _ in allres for f in fs]
        print(json.dumps({"world": dist.get_world_size(), "passed": total_pass, "failed": len(all_fail),
                          "onebit_bit_exact": sum(e for _, _, _, e in allres),
                          "launches": [l for _, _, l, _ in allres], "seconds": round(time.time() - t0, 1),
                          "failures": all_fail[:40]}))
    ok = all(not fs for _, fs, _, _ in allres)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
