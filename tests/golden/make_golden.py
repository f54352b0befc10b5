#!/usr/bin/env python3
"""Regenerate tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run in the authoring container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py

Every vector is produced by the reference library itself -- its own input
generators (std::mt19937 + uniform/normal distributions, exactly as in
tests/test_codec.cpp:53-60 and tests/test_collectives.cpp:41-47) and its own
Codec / c_fp_s / c_lp_s / d_fp_s / d_lp_s / Topology driven through its
SimCluster harness.  The fixtures travel with the repo; nothing at test time
reads /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402


def main():
    ref = Reference()
    out = {}

    # ---------------- codec: test_kernels.cpp kSizes x random_vec(-10,10), plus KAT inputs
    cases = []
    sizes = [1, 3, 7, 8, 9, 15, 16, 17, 64, 1000, 4097]
    for n in sizes:
        cases.append(ref.random_uniform(11 + n, n, -10.0, 10.0))
    for trial in range(30):  # test_codec.cpp:135-150 shapes
        cases.append(ref.random_uniform(100 + trial, 1 + trial * 7, -50.0, 50.0))
    cases += [np.array(v, np.float32) for v in ([-1.0, 1.0, 0.0], [0.0, 1.0, 0.5], [3.25, 3.25, 3.25],
                                               [0.0, -0.0, 1.0, -0.0], [-0.0, 0.0, -0.0],
                                               [1e-30, 2e-30, -3e-30], [3e38, -3e38, 0.0])]
    codec = {"count": np.array(len(cases))}
    for i, x in enumerate(cases):
        wire = ref.encode(x)
        codec[f"x{i}"] = x
        codec[f"wire{i}"] = wire
        codec[f"dec{i}"] = ref.decode(wire, x.size)
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), **codec)

    # ---------------- compensate_encode (uniform8), test_codec.cpp:230-244 shapes
    comp = {"count": np.array(20)}
    for t in range(20):
        x = ref.random_uniform(900 + t, 33, -5.0, 5.0)
        d = ref.random_uniform(950 + t, 33, -0.5, 0.5)
        d_in = d.copy()
        wire, dec = ref.compensate_encode(x, d)
        comp.update({f"x{t}": x, f"delta_in{t}": d_in, f"delta_out{t}": d, f"wire{t}": wire, f"dec{t}": dec})
    np.savez_compressed(os.path.join(HERE, "compensate_golden.npz"), **comp)

    # ---------------- collectives: test_collectives.cpp random_vec (normal), small shapes
    coll = {}
    idx = 0
    meta = []
    for g in (1, 2, 3, 4, 8):
        for n in (1, 5, 37, 1000):
            xs = [ref.random_normal(100 * g + r + 7 * n, n) for r in range(g)]
            rec = {"g": g, "n": n, "id": idx}
            for name in ("c_fp_s", "c_lp_s_u8", "c_lp_s_id", "d_fp_s_ring", "d_lp_s_ring", "d_fp_s_full_sum",
                         "d_lp_s_random"):
                ys = [x.copy() for x in xs]
                if name == "c_fp_s":
                    ref.c_fp_s(ys)
                elif name == "c_lp_s_u8":
                    ref.c_lp_s(ys, codec=1)
                elif name == "c_lp_s_id":
                    ref.c_lp_s(ys, codec=0)
                elif name == "d_fp_s_ring":
                    ref.d_fp_s(ys, topo_kind=0, seed=0, round_=3, mode=1)
                elif name == "d_lp_s_ring":
                    ref.d_lp_s(ys, topo_kind=0, seed=0, round_=3, codec=1, mode=1)
                elif name == "d_fp_s_full_sum":
                    ref.d_fp_s(ys, topo_kind=2, seed=0, round_=0, mode=0)
                elif name == "d_lp_s_random":
                    ref.d_lp_s(ys, topo_kind=1, seed=77, round_=5, codec=1, mode=1)
                coll[f"{idx}_{name}"] = np.stack(ys)
            coll[f"{idx}_in"] = np.stack(xs)
            meta.append(rec)
            idx += 1
    coll["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "collectives_golden.npz"), **coll)

    # ---------------- acceptance c4 shape: C_LP_S uint8 + EC, n=2, len=37, rounds traced
    g, n, rounds = 2, 37, 40
    ec = {}
    deltas = [np.zeros(n, np.float32) for _ in range(g)]
    eps = [np.zeros(len_, np.float32) for len_ in (19, 18)]
    for t in range(rounds):
        grads = [ref.random_uniform(7000 + 1000 * r + t, n, -1.0, 1.0) for r in range(g)]
        xs = [x.copy() for x in grads]
        ref.c_lp_s(xs, codec=1, deltas=deltas, eps=eps)
        ec[f"g{t}"] = np.stack(grads)
        ec[f"x{t}"] = np.stack(xs)
        ec[f"delta{t}"] = np.stack(deltas)
        ec[f"eps0_{t}"] = eps[0].copy()
        ec[f"eps1_{t}"] = eps[1].copy()
    ec["rounds"] = np.array(rounds)
    np.savez_compressed(os.path.join(HERE, "ec_trace_golden.npz"), **ec)

    # ---------------- topology: the random matching depends on libstdc++'s shuffle
    topo = {"random": {}, "ring": {}, "full": {}}
    for n in (1, 2, 3, 5, 8):
        for seed in (0, 123, 77):
            for rnd in range(6):
                for r in range(n):
                    topo["random"][f"{n},{seed},{rnd},{r}"] = ref.neighbors(1, n, seed, r, rnd)
        for r in range(n):
            topo["ring"][f"{n},{r}"] = ref.neighbors(0, n, 0, r, 0)
            topo["full"][f"{n},{r}"] = ref.neighbors(2, n, 0, r, 0)
    with open(os.path.join(HERE, "topology_golden.json"), "w") as f:
        json.dump(topo, f, indent=0, sort_keys=True)

    # ---------------- synthetic generator pin (host == device formula)
    syn = {f"seed{s}": ref.synth(4096, s) for s in (2026, 2027, 7)}
    np.savez_compressed(os.path.join(HERE, "synth_golden.npz"), **syn)
    print("golden fixtures written to", HERE, "backend", ref.backend())


if __name__ == "__main__":
    main()
