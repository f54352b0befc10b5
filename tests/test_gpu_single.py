"""GPU parity of the primitives at world size 1 (one GPU), through the C ABI.

g = 1 still runs the whole C_LP_S pipeline (both quantizations,
collectives.cpp:89-90); C_FP_S leaves x untouched (collectives.cpp:49);
D_* reduce over the singleton neighbourhood.  Bit-exact against the oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2107_01499_b200 as b2  # noqa: E402


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def ep():
    e = b2.B200Endpoint(0, 1, 0)
    yield e
    e.close()


U8 = b2.Codec(b2.CodecKind.uniform8)
ID = b2.Codec(b2.CodecKind.identity)


@pytest.mark.parametrize("n", [1, 5, 37, 4096, 1_000_003, 4_000_000])
def test_c_lp_s_g1(ep, oracle, n):
    x = oracle.synth(n, 2026)
    want = x.copy()
    oracle.c_lp_s([want], codec=1)
    t = torch.as_tensor(x).cuda()
    b2.c_lp_s(ep, 0.0, t, U8, None)
    assert np.array_equal(bits(t.cpu().numpy()), bits(want))


def test_c_lp_s_g1_headline_100m(ep, oracle):
    """The headline bucket (BASELINE.json config 3, 100M fp32) at g = 1, bit-exact,
    stateless and with error feedback (two rounds, state carried)."""
    n = 100_000_000
    stream = torch.cuda.current_stream().cuda_stream
    t = torch.empty(n, device="cuda")
    b2._lib.check(b2.lib.b2_fill_synthetic(t.data_ptr(), n, 2026, 0, stream))
    want = oracle.synth(n, 2026)
    oracle.c_lp_s([want], codec=1)
    b2.c_lp_s(ep, 0.0, t, U8, None, bucket=100)
    assert np.array_equal(bits(t.cpu().numpy()), bits(want))
    es = b2.ErrorState(n, n)
    d_or, e_or = [np.zeros(n, np.float32)], [np.zeros(n, np.float32)]
    for r in range(2):
        b2._lib.check(b2.lib.b2_fill_synthetic(t.data_ptr(), n, 3030 + r, 0, stream))
        want = oracle.synth(n, 3030 + r)
        oracle.c_lp_s([want], codec=1, deltas=d_or, eps=e_or)
        b2.c_lp_s(ep, 0.0, t, U8, es, bucket=101)
        assert np.array_equal(bits(t.cpu().numpy()), bits(want)), r
        assert np.array_equal(bits(es.delta.cpu().numpy()), bits(d_or[0])), r
        assert np.array_equal(bits(es.epsilon.cpu().numpy()), bits(e_or[0])), r
    del t, es
    ep.release_bucket(100)
    ep.release_bucket(101)


def test_c_lp_s_g1_identity_and_ec(ep, oracle):
    n = 1001
    x = oracle.synth(n, 7)
    want = x.copy()
    oracle.c_lp_s([want], codec=0)
    t = torch.as_tensor(x).cuda()
    b2.c_lp_s(ep, 0.0, t, ID, None, bucket=3)
    assert np.array_equal(bits(t.cpu().numpy()), bits(want))
    # error feedback, several rounds, state carried on the device
    es = b2.ErrorState(n, n)
    d_or = [np.zeros(n, np.float32)]
    e_or = [np.zeros(n, np.float32)]
    for r in range(5):
        g = oracle.synth(n, 100 + r)
        w = g.copy()
        oracle.c_lp_s([w], codec=1, deltas=d_or, eps=e_or)
        t = torch.as_tensor(g).cuda()
        b2.c_lp_s(ep, 0.0, t, U8, es, bucket=4)
        assert np.array_equal(bits(t.cpu().numpy()), bits(w))
        assert np.array_equal(bits(es.delta.cpu().numpy()), bits(d_or[0]))
        assert np.array_equal(bits(es.epsilon.cpu().numpy()), bits(e_or[0]))


def test_c_fp_s_g1_untouched(ep):
    x = np.array([-0.0, 1.0, 2.5], np.float32)
    t = torch.as_tensor(x).cuda()
    b2.c_fp_s(ep, 0.0, t)
    assert np.array_equal(bits(t.cpu().numpy()), bits(x))


def test_d_primitives_g1(ep, oracle):
    n = 5003
    x = oracle.synth(n, 9)
    topo = b2.Topology(b2.TopologyKind.ring, 1, 0)
    for mode in (b2.ReduceMode.sum, b2.ReduceMode.average):
        t = torch.as_tensor(x).cuda()
        b2.d_fp_s(ep, 0.0, t, topo, 0, mode)
        assert np.array_equal(bits(t.cpu().numpy()), bits(oracle.d_fp_s_rank([x], int(mode))))
        t = torch.as_tensor(x).cuda()
        b2.d_lp_s(ep, 0.0, t, topo, 0, U8, mode)
        assert np.array_equal(bits(t.cpu().numpy()), bits(oracle.d_lp_s_rank([x], 1, int(mode))))


def test_nonfinite_bucket_raises(ep):
    x = torch.ones(1000, device="cuda")
    x[500] = float("nan")
    with pytest.raises(b2.Error):
        b2.c_lp_s(ep, 0.0, x, U8, None, bucket=9)
    y = torch.ones(1000, device="cuda")
    y[3] = float("inf")
    with pytest.raises(b2.Error):
        b2.d_lp_s(ep, 0.0, y, b2.Topology(b2.TopologyKind.ring, 1), 0, U8, b2.ReduceMode.average, bucket=9)


def test_argument_errors(ep):
    x = torch.ones(10, device="cuda")
    with pytest.raises(b2.Error):
        b2.c_lp_s(ep, 0.0, x, U8, b2.ErrorState(3, 1))  # collectives.cpp:102-107
    with pytest.raises(b2.Error):
        b2.d_fp_s(ep, 0.0, x, b2.Topology(b2.TopologyKind.full, 5), 0, b2.ReduceMode.sum)


def test_host_buffer_path(ep, oracle):
    x = oracle.synth(4099, 31)
    want = x.copy()
    oracle.c_lp_s([want], codec=1)
    y = x.copy()
    b2.c_lp_s(ep, 0.0, y, U8, None, bucket=11)  # numpy in place, staged through the GPU
    assert np.array_equal(bits(y), bits(want))
    # unpinned torch tensor: the same, through the cached pinned bounce buffer
    z = torch.as_tensor(x.copy())
    b2.c_lp_s(ep, 0.0, z, U8, None, bucket=11)
    assert np.array_equal(bits(z.numpy()), bits(want))


def test_host_pinned_pipeline(ep, oracle):
    """Pinned host buckets with blocking=False: uploads, kernels and downloads
    of consecutive calls overlap on the endpoint's copy streams; after
    ep.sync() every buffer holds its own call chain's result."""
    n = 1_000_003
    bufs = [torch.as_tensor(oracle.synth(n, 70 + b)).pin_memory() for b in range(3)]
    want = [oracle.synth(n, 70 + b) for b in range(3)]
    for i in range(9):
        b2.c_lp_s(ep, 0.0, bufs[i % 3], U8, None, bucket=12, blocking=False)
        w = [want[i % 3]]
        oracle.c_lp_s(w, codec=1)
    ep.sync()
    for b in range(3):
        assert np.array_equal(bits(bufs[b].numpy()), bits(want[b])), b


def test_host_nonfinite_leaves_x_untouched(ep):
    """The reference throws from encode before x changes (codec.cpp:24-27):
    a blocking host call checks the device status before writing back."""
    x = np.ones(5000, np.float32)
    x[17] = np.inf
    before = x.copy()
    with pytest.raises(b2.Error):
        b2.c_lp_s(ep, 0.0, x, U8, None, bucket=13)
    assert np.array_equal(bits(x), bits(before))
    p = torch.ones(5000).pin_memory()
    p[9] = float("nan")
    before = p.clone()
    with pytest.raises(b2.Error):
        b2.c_lp_s(ep, 0.0, p, U8, None, bucket=13)
    assert np.array_equal(bits(p.numpy()), bits(before.numpy()))


def test_flatten_aliasing_and_collective(ep, oracle):
    # test_tensor.cpp:10-60 on device memory, then a collective on the arena
    t1 = b2.FlatTensor("t1", [2], [1.0, 2.0])
    t2 = b2.FlatTensor("t2", [1], [3.0])
    arena = b2.BucketArena.flatten([t1, t2])
    assert arena.size() == 3 and arena.data().cpu().tolist() == [1.0, 2.0, 3.0]
    assert [(m.offset, m.length) for m in arena.members()] == [(0, 2), (2, 1)]
    arena.data()[2] = 9.0
    assert float(t2[0]) == 9.0
    t1[1] = -4.0
    assert float(arena.data()[1]) == -4.0
    flat = arena.as_flat()
    flat[0] = 11.0
    assert float(t1[0]) == 11.0
    with pytest.raises(b2.Error):
        b2.BucketArena.flatten([b2.FlatTensor("x", [1], [1.0]), b2.FlatTensor("x", [1], [2.0])])
    with pytest.raises(b2.Error):
        b2.BucketArena.flatten([])
    # many members (> one 64-member launch), then C_LP_S on the arena aliases back
    rng = np.random.default_rng(99)
    vals = [rng.uniform(-100, 100, int(rng.integers(1, 50))).astype(np.float32) for _ in range(150)]
    ts = [b2.FlatTensor(f"p{i}", [v.size], v) for i, v in enumerate(vals)]
    a = b2.BucketArena.flatten(ts)
    cat = np.concatenate(vals)
    assert np.array_equal(a.data().cpu().numpy(), cat)
    want = cat.copy()
    oracle.c_lp_s([want], codec=1)
    b2.c_lp_s(ep, 0.0, a, U8, None, bucket=12)
    off = 0
    for t, v in zip(ts, vals):
        assert np.array_equal(bits(t.data().cpu().numpy()), bits(want[off:off + v.size]))
        off += v.size


@pytest.mark.parametrize("case", ["constant", "two_levels", "tiny_range", "signed_zeros", "huge_finite",
                                  "overflow_range", "subnormal"])
def test_c_lp_s_g1_edge_inputs(ep, oracle, case):
    """Edge inputs for the single-rank path (its second header is derived
    from the first, so degenerate / extreme ranges are pinned explicitly)."""
    n = 4099
    rng = np.random.default_rng(7)
    x = {
        "constant": np.full(n, 3.25, np.float32),
        "two_levels": np.where(rng.random(n) < 0.5, -1.5, 2.0).astype(np.float32),
        "tiny_range": (1.0 + rng.random(n) * 1e-6).astype(np.float32),
        "signed_zeros": np.where(rng.random(n) < 0.5, 0.0, -0.0).astype(np.float32),
        "huge_finite": (rng.standard_normal(n) * 1e37).astype(np.float32),
        "overflow_range": np.where(rng.random(n) < 0.5, -3e38, 3e38).astype(np.float32),
        "subnormal": (rng.standard_normal(n) * 1e-40).astype(np.float32),
    }[case]
    want = x.copy()
    try:
        oracle.c_lp_s([want], codec=1)
        ref_err = False
    except ValueError:
        ref_err = True
    t = torch.as_tensor(x).cuda()
    if ref_err:
        with pytest.raises(b2.Error):
            b2.c_lp_s(ep, 0.0, t, U8, None, bucket=20)
    else:
        b2.c_lp_s(ep, 0.0, t, U8, None, bucket=20)
        assert np.array_equal(bits(t.cpu().numpy()), bits(want))


# ---------------------------------------------------------- C_LP_S onebit
OB = b2.Codec(b2.CodecKind.onebit)


def test_c_lp_s_onebit_reference_kat(ep):
    # test_collectives.cpp:209-225: single-worker sign compression with EC
    t = torch.tensor([0.3, -0.1], dtype=torch.float32).cuda()
    es = b2.ErrorState(2, 2)
    b2.c_lp_s(ep, 0.0, t, OB, es, bucket=40)
    x, d, e = t.cpu().numpy(), es.delta.cpu().numpy(), es.epsilon.cpu().numpy()
    assert x[0] == pytest.approx(0.2) and x[1] == pytest.approx(-0.2)
    assert d[0] == pytest.approx(0.1, rel=1e-6) and d[1] == pytest.approx(0.1, rel=1e-6)
    assert e[0] == pytest.approx(0.0) and e[1] == pytest.approx(0.0)


@pytest.mark.parametrize("n", [1, 5, 37, 1023, 1025, 4096, 1_000_003, 4_000_000])
def test_c_lp_s_onebit_g1(ep, oracle, n):
    # splitmix grid inputs: every fp64 |x| sum is exact, so bit-exact
    x = oracle.synth(n, 3030 + n)
    want = x.copy()
    oracle.c_lp_s([want], codec=2)
    t = torch.as_tensor(x).cuda()
    b2.c_lp_s(ep, 0.0, t, OB, None, bucket=41)
    assert np.array_equal(bits(t.cpu().numpy()), bits(want))


def test_c_lp_s_onebit_g1_ec_rounds(ep, oracle):
    # y = x - delta makes the |y| sums inexact: scales within a float
    # rounding of the oracle's (sequential fp64, as the reference's scalar path)
    n = 100_003
    es = b2.ErrorState(n, n)
    d_or, e_or = [np.zeros(n, np.float32)], [np.zeros(n, np.float32)]
    for r in range(6):
        g = oracle.synth(n, 400 + r)
        w = g.copy()
        oracle.c_lp_s([w], codec=2, deltas=d_or, eps=e_or)
        t = torch.as_tensor(g).cuda()
        b2.c_lp_s(ep, 0.0, t, OB, es, bucket=42)
        for got, want in ((t, w), (es.delta, d_or[0]), (es.epsilon, e_or[0])):
            tol = 4 * np.spacing(np.float32(np.abs(want).max()))
            assert np.abs(got.cpu().numpy() - want).max() <= tol


def test_c_lp_s_onebit_nonfinite_raises(ep):
    t = torch.tensor([1.0, float("inf"), 2.0], dtype=torch.float32).cuda()
    with pytest.raises(b2.Error):
        b2.c_lp_s(ep, 0.0, t, OB, None, bucket=43)


@pytest.mark.parametrize("n", [1, 37, 1025, 1_000_003])
def test_d_lp_s_onebit_g1(ep, oracle, n):
    x = oracle.synth(n, 5050 + n)
    topo = b2.Topology(b2.TopologyKind.ring, 1)
    for mode in (b2.ReduceMode.average, b2.ReduceMode.sum):
        t = torch.as_tensor(x).cuda()
        b2.d_lp_s(ep, 0.0, t, topo, 0, OB, mode, bucket=44)
        assert np.array_equal(bits(t.cpu().numpy()), bits(oracle.d_lp_s_rank([x], 2, int(mode))))


def test_engine_reports_nonfinite_gradient(oracle):
    """OverlapEngine.finish() is non-blocking; a non-finite gradient of its
    buckets (the reference throws from encode, codec.cpp:24-27) is raised by
    synchronize(), or by the next finish() once those buckets completed."""
    from paper_2107_01499_b200.engine import OverlapEngine
    ep = b2.B200Endpoint(0, 1, 0)
    eng = OverlapEngine(ep, [1000, 3000, 500], capacity_bytes=4 * 2000, sm_budget=32)
    for layer in reversed(range(3)):
        eng.grad(layer).copy_(torch.as_tensor(oracle.synth(eng.sizes[layer], 40 + layer)))
        if layer == 1:
            eng.grad(layer)[7] = float("nan")
        eng.layer_done(layer)
    eng.finish()
    with pytest.raises(b2.Error):
        eng.synchronize()
    # a clean iteration afterwards works (a non-finite input does not poison)
    for layer in reversed(range(3)):
        eng.grad(layer).copy_(torch.as_tensor(oracle.synth(eng.sizes[layer], 50 + layer)))
        eng.layer_done(layer)
    eng.finish()
    eng.synchronize()
    for bk in eng.buckets:
        xs = [np.concatenate([oracle.synth(eng.sizes[l], 50 + l) for l in bk.layers])]
        oracle.c_lp_s(xs, codec=1)
        assert np.array_equal(bits(eng.arenas[bk.id].cpu().numpy()), bits(xs[0]))
    ep.close()


def test_c_lp_s_stochastic_g1_unbiased(ep):
    """Codec{uniform8, Rounding::stochastic} inside C_LP_S and D_LP_S
    (codec.cpp:67-78): every encode rounds stochastically; the expected output
    equals the input (test_codec.cpp:175-192's unbiasedness), outputs lie on
    the 1/255 grid of the headers (0, 1), the same generator state gives the
    same result and the generator advances per call."""
    import random
    st = b2.Codec(b2.CodecKind.uniform8, b2.Rounding.stochastic)
    n = 200_000
    x = np.full(n, 0.3777, np.float32)
    x[0], x[1] = 0.0, 1.0
    for prim in ("c_lp_s", "d_lp_s"):
        rng = random.Random(3)
        outs = []
        for _ in range(2):
            t = torch.as_tensor(x).cuda()
            if prim == "c_lp_s":
                b2.c_lp_s(ep, 0.0, t, st, None, rng, bucket=40)
            else:
                b2.d_lp_s(ep, 0.0, t, b2.Topology(b2.TopologyKind.ring, 1), 0, st, b2.ReduceMode.average, rng,
                          bucket=41)
            outs.append(t.cpu().numpy())
        y = outs[0].astype(np.float64)
        assert y[0] == 0.0 and y[1] == 1.0
        lv = np.round(y * 255.0)
        assert np.all(np.abs(y - lv / 255.0) < 1e-6)  # on the grid
        e = y[2:] - np.float64(np.float32(0.3777))
        assert abs(e.mean()) <= 4.0 * np.sqrt(e.var() / e.size), (prim, e.mean())
        assert not np.array_equal(outs[0], outs[1])  # the generator advanced
        t = torch.as_tensor(x).cuda()
        if prim == "c_lp_s":
            b2.c_lp_s(ep, 0.0, t, st, None, random.Random(3), bucket=40)
        else:
            b2.d_lp_s(ep, 0.0, t, b2.Topology(b2.TopologyKind.ring, 1), 0, st, b2.ReduceMode.average,
                      random.Random(3), bucket=41)
        assert np.array_equal(t.cpu().numpy(), outs[0])  # same stream, same draws
    with pytest.raises(b2.Error):
        b2.c_lp_s(ep, 0.0, torch.as_tensor(x).cuda(), st, None, None)  # codec.cpp:68-70


def test_hierarchical_c_one_rank_c_abi(ep, oracle):
    """b2_hierarchical_c over one node with one rank: the reference's member
    fold (float)(0.0 + (double)x) (collectives.cpp:321-332, 377-380), so -0.0
    becomes +0.0 and every other value is unchanged."""
    x = oracle.synth(4099, 12)
    x[::7] = -0.0
    want = x.copy()
    oracle.hierarchical_c([want], [0], 1)
    t = torch.as_tensor(x).cuda()
    b2._lib.check(b2.lib.b2_hierarchical_c(ep.handle, t.data_ptr(), t.numel(), 50,
                                           torch.cuda.current_stream().cuda_stream))
    ep.sync()
    assert np.array_equal(bits(t.cpu().numpy()), bits(want))
    assert not np.signbit(t.cpu().numpy()[0])
