"""Live cross-check of the C restatement against the compiled reference
(oracle/_ref), on inputs the fixtures do not cover.  Skipped where the
reference library was not built (it is built from /root/reference)."""
import numpy as np
import pytest


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("g", [1, 2, 3, 8])
@pytest.mark.parametrize("n", [5, 37, 100_003])
def test_c_primitives_match_reference(oracle, ref, g, n):
    xs = [ref.synth(n, 2026 + r) for r in range(g)]
    for codec in (0, 1):
        a = [x.copy() for x in xs]
        b = [x.copy() for x in xs]
        oracle.c_lp_s(a, codec=codec)
        ref.c_lp_s(b, codec=codec)
        assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(a, b))
    a = [x.copy() for x in xs]
    b = [x.copy() for x in xs]
    oracle.c_fp_s(a)
    ref.c_fp_s(b)
    assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(a, b))


@pytest.mark.parametrize("g", [2, 4, 8])
def test_d_primitives_match_reference(oracle, ref, g):
    n = 50_001
    xs = [ref.synth(n, 99 + r) for r in range(g)]
    for kind, seed in ((0, 0), (1, 5), (2, 0)):
        for mode in (0, 1):
            b = [x.copy() for x in xs]
            ref.d_lp_s(b, topo_kind=kind, seed=seed, round_=2, codec=1, mode=mode)
            c = [x.copy() for x in xs]
            ref.d_fp_s(c, topo_kind=kind, seed=seed, round_=2, mode=mode)
            for r in range(g):
                nb = ref.neighbors(kind, g, seed, r, 2)
                assert np.array_equal(bits(oracle.d_lp_s_rank([xs[j] for j in nb], 1, mode)), bits(b[r]))
                assert np.array_equal(bits(oracle.d_fp_s_rank([xs[j] for j in nb], mode)), bits(c[r]))


def test_ec_rounds_match_reference(oracle, ref):
    g, n = 3, 1001
    da = [np.zeros(n, np.float32) for _ in range(g)]
    db = [np.zeros(n, np.float32) for _ in range(g)]
    ea = [np.zeros(oracle.partition_range(n, g, r)[1], np.float32) for r in range(g)]
    eb = [e.copy() for e in ea]
    for t in range(5):
        xs = [ref.synth(n, 500 + 10 * t + r) for r in range(g)]
        a = [x.copy() for x in xs]
        b = [x.copy() for x in xs]
        oracle.c_lp_s(a, codec=1, deltas=da, eps=ea)
        ref.c_lp_s(b, codec=1, deltas=db, eps=eb)
        assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(a, b))
        assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(da, db))
        assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(ea, eb))


def test_wire_counts_match_reference(ref):
    # bytes on the wire per worker: 2(g-1)/g * 4N for c_fp_s
    g, n = 8, 80_000
    xs = [ref.synth(n, r) for r in range(g)]
    b, m = ref.c_fp_s([x.copy() for x in xs])
    assert all(v == 2 * (g - 1) for v in m)
    assert all(v == 4 * n * 2 * (g - 1) // g for v in b)
    bl = ref.c_lp_s([x.copy() for x in xs], codec=1)
    assert all(v == 2 * (g - 1) * (8 + n // g) for v in bl)


@pytest.mark.parametrize("n", [1, 3, 8, 9, 37, 100_003])
def test_onebit_codec_matches_reference(oracle, ref, n):
    # codec.cpp:81-88, 110-114: sign bytes bit-exact; the scale from the
    # reference's active backend (AVX2 sums |x| in 4 fp64 lanes, the scalar
    # path sequentially) equals the oracle's (sequential) exactly when the
    # fp64 sum is exact -- always for the splitmix grid inputs -- and within
    # one float rounding for gaussians
    x = ref.synth(n, 77 + n)
    w_ref = ref.encode(x, codec=2)
    w_orc = oracle.onebit_encode_wire(x)
    assert np.array_equal(w_ref, w_orc)
    assert np.array_equal(bits(ref.decode(w_ref, n, codec=2)), bits(oracle.onebit_decode_wire(w_orc, n)))
    g = ref.random_normal(n, 5 + n) if hasattr(ref, "random_normal") else x
    a, b = ref.encode(g, codec=2), oracle.onebit_encode_wire(g)
    assert np.array_equal(a[4:], b[4:])
    sa, sb = a[:4].view(np.float32)[0], b[:4].view(np.float32)[0]
    assert abs(sa - sb) <= np.spacing(np.float32(max(abs(sa), abs(sb))))


def test_onebit_reference_kats(oracle):
    # test_codec.cpp:103-132, transcribed
    w = oracle.onebit_encode_wire(np.array([1, -1, 1, 1, -1, 1, 1, 1, -1], np.float32))
    assert w[:4].view(np.float32)[0] == 1.0 and w[4] == 0b11101101 and w[5] == 0
    assert list(oracle.onebit_decode_wire(oracle.onebit_encode_wire(np.array([1, -2, 3], np.float32)), 3)) == \
        [2.0, -2.0, 2.0]
    assert list(oracle.onebit_decode_wire(oracle.onebit_encode_wire(np.array([-1, -3], np.float32)), 2)) == \
        [-2.0, -2.0]


@pytest.mark.parametrize("g", [1, 2, 3, 8])
@pytest.mark.parametrize("n", [5, 37, 100_003])
def test_onebit_c_lp_s_matches_reference(oracle, ref, g, n):
    # c_lp_s with Codec{onebit} (the 1-bit Adam aggregation, algorithms.cpp:
    # 141-148).  Without EC on splitmix grid inputs every fp64 |x| sum is
    # exact, so the restatement must be bitwise equal to the reference.
    xs = [ref.synth(n, 4040 + r) for r in range(g)]
    a = [x.copy() for x in xs]
    b = [x.copy() for x in xs]
    oracle.c_lp_s(a, codec=2)
    ref.c_lp_s(b, codec=2)
    assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(a, b))


def test_onebit_ec_rounds_match_reference(oracle, ref):
    # with error feedback the |y| sums stop being exact (y = x - delta), so
    # the scales agree within a float rounding: values within 4 ulp of the
    # reference's scale magnitude, residual state likewise
    g, n = 3, 1001
    da = [np.zeros(n, np.float32) for _ in range(g)]
    db = [np.zeros(n, np.float32) for _ in range(g)]
    ea = [np.zeros(oracle.partition_range(n, g, r)[1], np.float32) for r in range(g)]
    eb = [e.copy() for e in ea]
    for t in range(5):
        xs = [ref.synth(n, 700 + 10 * t + r) for r in range(g)]
        a = [x.copy() for x in xs]
        b = [x.copy() for x in xs]
        oracle.c_lp_s(a, codec=2, deltas=da, eps=ea)
        ref.c_lp_s(b, codec=2, deltas=db, eps=eb)
        for p, q in zip(a + da + ea, b + db + eb):
            tol = 4 * np.spacing(np.float32(np.abs(q).max() if q.size else 1.0))
            assert np.abs(p - q).max(initial=0) <= tol


@pytest.mark.parametrize("g", [2, 4, 8])
def test_onebit_d_lp_s_matches_reference(oracle, ref, g):
    # d_lp_s with Codec{onebit} (collectives.cpp:260-288); grid inputs: exact sums, bitwise
    n = 50_001
    xs = [ref.synth(n, 1313 + r) for r in range(g)]
    for kind, seed in ((0, 0), (1, 5), (2, 0)):
        for mode in (0, 1):
            b = [x.copy() for x in xs]
            ref.d_lp_s(b, topo_kind=kind, seed=seed, round_=1, codec=2, mode=mode)
            for r in range(g):
                nb = ref.neighbors(kind, g, seed, r, 1)
                assert np.array_equal(bits(oracle.d_lp_s_rank([xs[j] for j in nb], 2, mode)), bits(b[r]))


@pytest.mark.parametrize("nodes", [[0, 0, 0, 1, 1, 2], [0, 0, 1, 1], [0, 1], [0, 0, 0], [2, 0, 1, 0, 2, 1, 1, 0]])
@pytest.mark.parametrize("codec", [0, 1, 2])
def test_hierarchical_c_matches_reference(oracle, ref, nodes, codec):
    # collectives.cpp:290-385: intra-node fp64 sum at the leader, leaders
    # exchange fp64 partials (lossless) or run scatter_reduce_lp, members get
    # the leader's result; the restatement must be bitwise equal
    g, n = len(nodes), 10_007
    xs = [ref.synth(n, 5150 + r) for r in range(g)]
    a = [x.copy() for x in xs]
    b = [x.copy() for x in xs]
    oracle.hierarchical_c(a, nodes, codec)
    ref.hierarchical_c(b, nodes, codec)
    assert all(np.array_equal(bits(p), bits(q)) for p, q in zip(a, b))
