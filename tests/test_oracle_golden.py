"""Pin the CPU oracle (oracle/rcomm_oracle.c) to the reference: its own
known-answer tests (tests/golden/kats.json, with file:line) and fixtures the
unmodified reference produced (tests/golden/*.npz, make_golden.py).
CPU only -- this is what makes the oracle trustworthy as the GPU checker."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        return json.load(f)


def test_kat_wire(oracle, kats):
    k = kats["wire_u8"]
    w = oracle.encode_wire(np.array(k["x"], np.float32))
    assert w.size == k["payload_size"]
    assert w[:4].view(np.float32)[0] == k["min"] and w[4:8].view(np.float32)[0] == k["max"]
    assert list(w[8:]) == k["codes"]


def test_kat_endpoints_degenerate(oracle, kats):
    lo, hi, c = oracle.encode(np.array(kats["endpoints"]["x"], np.float32))
    assert list(oracle.decode(lo, hi, c)) == kats["endpoints"]["decoded"]
    lo, hi, c = oracle.encode(np.array(kats["endpoints"]["mid_x"], np.float32))
    assert c[2] == kats["endpoints"]["mid_level"]
    lo, hi, c = oracle.encode(np.array(kats["degenerate"]["x"], np.float32))
    assert list(oracle.decode(lo, hi, c)) == kats["degenerate"]["decoded"]


def test_kat_quantize_minmax(oracle, kats):
    k = kats["quantize_rne_clamp"]
    assert list(oracle.quantize_u8(np.array(k["x"], np.float32), k["min"], k["inv_step"])) == k["codes"]
    k = kats["minmax"]
    assert oracle.minmax(np.array(k["x"], np.float32)) == (k["min"], k["max"])


def test_kat_nonfinite(oracle):
    for bad in ([1.0, np.inf], [np.nan], [-np.inf, 1.0]):
        with pytest.raises(ValueError):
            oracle.encode(np.array(bad, np.float32))


def test_kat_partition_and_topology(oracle, kats):
    for n, g, k, lo, sz in kats["partition_range"]["cases"]:
        assert oracle.partition_range(n, g, k) == (lo, sz)
    for n, w, i, own in kats["partition_range"]["owned"]:
        assert oracle.partition_range(n, w, i)[1] == own
    t = kats["topology"]
    assert oracle.neighbors(1, 4, 0) == t["ring4"]["0,0"]
    assert oracle.neighbors(1, 4, 2) == t["ring4"]["2,7"]
    assert oracle.neighbors(1, 2, 0) == t["ring2"]["0,0"]
    assert oracle.neighbors(1, 1, 0) == t["ring1"]["0,0"]
    assert oracle.neighbors(2, 3, 1) == t["full3"]["1,5"]
    with pytest.raises(ValueError):
        oracle.neighbors(1, 4, 4)


def test_kat_ring_average_and_sum(oracle, kats):
    xs = [np.array(v, np.float32) for v in kats["ring_average"]["xs"]]
    for r in range(4):
        nb = oracle.neighbors(1, 4, r)
        got = oracle.d_fp_s_rank([xs[j] for j in nb], 1)
        assert abs(got[0] - kats["ring_average"]["approx"][r]) < 1e-6
    xs = [np.array(v, np.float32) for v in kats["sum_mode"]["xs"]]
    for r in range(3):
        assert oracle.d_fp_s_rank(xs, 0)[0] == kats["sum_mode"]["sum"]


def test_codec_fixtures(oracle):
    z = np.load(os.path.join(GOLDEN, "codec_golden.npz"))
    for i in range(int(z["count"])):
        x, wire = z[f"x{i}"], z[f"wire{i}"]
        w = oracle.encode_wire(x)
        assert np.array_equal(w[8:], wire[8:]), i
        # +-0 ties compare with == (test_kernels.cpp:111)
        assert w[:4].view(np.float32)[0] == wire[:4].view(np.float32)[0]
        assert w[4:8].view(np.float32)[0] == wire[4:8].view(np.float32)[0]
        lo, hi = wire[:4].view(np.float32)[0], wire[4:8].view(np.float32)[0]
        assert np.array_equal(bits(oracle.decode(lo, hi, wire[8:])), bits(z[f"dec{i}"])), i


def test_compensate_fixtures(oracle):
    z = np.load(os.path.join(GOLDEN, "compensate_golden.npz"))
    for t in range(int(z["count"])):
        d = z[f"delta_in{t}"].copy()
        lo, hi, codes, dec = oracle.compensate_encode(z[f"x{t}"], d)
        assert np.array_equal(codes, z[f"wire{t}"][8:])
        assert np.array_equal(bits(d), bits(z[f"delta_out{t}"]))
        assert np.array_equal(bits(dec), bits(z[f"dec{t}"]))


def test_collective_fixtures(oracle):
    z = np.load(os.path.join(GOLDEN, "collectives_golden.npz"))
    with open(os.path.join(GOLDEN, "topology_golden.json")) as f:
        topo = json.load(f)
    for rec in json.loads(str(z["meta"])):
        g, n, i = rec["g"], rec["n"], rec["id"]
        xs = list(z[f"{i}_in"])
        ys = [x.copy() for x in xs]
        oracle.c_fp_s(ys)
        assert np.array_equal(bits(np.stack(ys)), bits(z[f"{i}_c_fp_s"])), (g, n)
        ys = [x.copy() for x in xs]
        oracle.c_lp_s(ys, codec=1)
        assert np.array_equal(bits(np.stack(ys)), bits(z[f"{i}_c_lp_s_u8"])), (g, n)
        ys = [x.copy() for x in xs]
        oracle.c_lp_s(ys, codec=0)
        assert np.array_equal(bits(np.stack(ys)), bits(z[f"{i}_c_lp_s_id"])), (g, n)
        for r in range(g):
            nb = oracle.neighbors(1, g, r)
            assert np.array_equal(bits(oracle.d_fp_s_rank([xs[j] for j in nb], 1)), bits(z[f"{i}_d_fp_s_ring"][r]))
            assert np.array_equal(bits(oracle.d_lp_s_rank([xs[j] for j in nb], 1, 1)),
                                  bits(z[f"{i}_d_lp_s_ring"][r]))
            assert np.array_equal(bits(oracle.d_fp_s_rank(xs, 0)), bits(z[f"{i}_d_fp_s_full_sum"][r]))
            nbr = topo["random"][f"{g},77,5,{r}"] if f"{g},77,5,{r}" in topo["random"] else None
            if nbr is not None:
                assert np.array_equal(bits(oracle.d_lp_s_rank([xs[j] for j in nbr], 1, 1)),
                                      bits(z[f"{i}_d_lp_s_random"][r]))


def test_ec_trace_fixture(oracle):
    # acceptance.cpp:255-350 shape: 2 workers, 37 elements, error feedback carried
    z = np.load(os.path.join(GOLDEN, "ec_trace_golden.npz"))
    deltas = [np.zeros(37, np.float32) for _ in range(2)]
    eps = [np.zeros(19, np.float32), np.zeros(18, np.float32)]
    for t in range(int(z["rounds"])):
        xs = [x.copy() for x in z[f"g{t}"]]
        oracle.c_lp_s(xs, codec=1, deltas=deltas, eps=eps)
        assert np.array_equal(bits(np.stack(xs)), bits(z[f"x{t}"])), t
        assert np.array_equal(bits(np.stack(deltas)), bits(z[f"delta{t}"])), t
        assert np.array_equal(bits(eps[0]), bits(z[f"eps0_{t}"])) and np.array_equal(bits(eps[1]), bits(z[f"eps1_{t}"]))


def test_synth_fixture(oracle):
    z = np.load(os.path.join(GOLDEN, "synth_golden.npz"))
    for s in (2026, 2027, 7):
        assert np.array_equal(bits(oracle.synth(4096, s)), bits(z[f"seed{s}"]))
    # partition-local generation (offset) == slice of the full stream
    full = oracle.synth(10_000, 5)
    assert np.array_equal(bits(oracle.synth(1000, 5, 4321)), bits(full[4321:5321]))


def test_oracle_properties(oracle):
    """Size-independent properties at sizes beyond the fixtures."""
    rng = np.random.default_rng(0)
    for n in (1, 17, 100_000):
        x = (rng.standard_normal(n) * 3).astype(np.float32)
        lo, hi, c = oracle.encode(x)
        y = oracle.decode(lo, hi, c)
        step = (float(hi) - float(lo)) / 255.0
        err = np.abs(y.astype(np.float64) - x)
        assert np.all(err <= step * (1 + 1e-5))  # acceptance.cpp:197-214 (one step)
        slack = 2.0 ** -21 * max(abs(float(lo)), abs(float(hi)))  # fp32 rounding of lo + q*step
        assert np.all(err <= step / 2 + slack)  # test_codec.cpp:152-166 (half step, nearest)
