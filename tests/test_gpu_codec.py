"""GPU parity: the uniform8 codec kernels vs the oracle / the reference's KATs.

Bar: codes bit-exact; (min, max) bit-exact with +-0 compared
by ==; decoded fp32 bit-exact (no FMA, same rounding) -- stricter than the
north_star floor of one quantization step.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2107_01499_b200 as b2  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U8 = b2.Codec(b2.CodecKind.uniform8)


def dev(a):
    return torch.as_tensor(np.asarray(a, np.float32)).cuda()


def enc(x):
    codes, hdr = U8.encode_soa(dev(x))
    return codes.cpu().numpy(), hdr[:2].cpu().numpy()


def bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def same(a, b):
    """Bit-identical, except that NaN payloads compare equal: IEEE 754 leaves
    them unspecified and x86 (0xffc00000) and CUDA (0x7fffffff) differ."""
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    return a.shape == b.shape and bool(np.all((bits(a) == bits(b)) | (np.isnan(a) & np.isnan(b))))


def test_wire_kat():
    # test_codec.cpp:114-123
    p = U8.encode(dev([-1.0, 1.0, 0.0])).cpu().numpy()
    assert p.size == 11
    assert p[:4].view(np.float32)[0] == -1.0 and p[4:8].view(np.float32)[0] == 1.0
    assert list(p[8:]) == [0, 255, 128]


def test_endpoints_and_midpoint():
    # test_codec.cpp:82-94
    y = U8.decode(U8.encode(dev([0.0, 1.0])), 2).cpu().numpy()
    assert y[0] == 0.0 and y[1] == 1.0
    z = U8.decode(U8.encode(dev([0.0, 1.0, 0.5])), 3).cpu().numpy()
    assert abs(z[2] - 128.0 / 255.0) <= 1e-6 * 128.0 / 255.0


def test_degenerate_constant():
    # test_codec.cpp:96-101
    y = U8.decode(U8.encode(dev([3.25, 3.25, 3.25])), 3).cpu().numpy()
    assert (y == 3.25).all()


def test_quantize_rne_and_clamp_kat():
    # test_kernels.cpp:131-142 drives quantize_u8 with (min=0, inv_step=1).  Through
    # the codec the same levels appear with min=0, max=255 (inv_step = 1 exactly).
    x = [0.0, 255.0, 0.5, 1.5, 2.5, 254.49]
    codes, hdr = enc(x)
    assert list(hdr) == [0.0, 255.0]
    assert list(codes) == [0, 255, 0, 2, 2, 254]


def test_nonfinite_raises():
    # test_codec.cpp:247-253
    with pytest.raises(b2.Error):
        U8.encode(dev([1.0, np.inf]))
    with pytest.raises(b2.Error):
        U8.encode(dev([np.nan]))
    with pytest.raises(b2.Error):
        U8.encode(dev([-np.inf, 2.0, 3.0, 4.0, 5.0]))
    with pytest.raises(b2.Error):
        U8.decode(torch.tensor([1, 2, 3], dtype=torch.uint8).cuda(), 10)


def test_stochastic_rounding_needs_a_generator():
    with pytest.raises(b2.Error):  # codec.cpp:70
        b2.Codec(b2.CodecKind.uniform8, b2.Rounding.stochastic).encode(dev([1.0, 2.0]))


# ------------------------------------------------------------------ onebit
OB = b2.Codec(b2.CodecKind.onebit)


def test_onebit_kats():
    # test_codec.cpp:103-132
    w = OB.encode(np.array([1, -1, 1, 1, -1, 1, 1, 1, -1], np.float32))
    assert len(w) == 6 and w[:4].view(np.float32)[0] == 1.0 and w[4] == 0b11101101 and w[5] == 0
    assert list(OB.decode(OB.encode(np.array([1, -2, 3], np.float32)), 3)) == [2.0, -2.0, 2.0]
    assert list(OB.decode(OB.encode(np.array([-1, -3], np.float32)), 2)) == [-2.0, -2.0]
    w0 = OB.encode(np.zeros(0, np.float32))
    assert len(w0) == 4 and w0.view(np.float32)[0] == 0.0
    with pytest.raises(b2.Error):
        OB.encode(dev([1.0, float("inf")]))
    with pytest.raises(b2.Error):
        OB.encode(dev([float("nan")] * 40))


@pytest.mark.parametrize("n", [1, 3, 31, 32, 33, 64, 1000, 4097, 100_003, 4_000_000])
def test_onebit_vs_oracle(oracle, n):
    # splitmix grid inputs: the fp64 |x| sum is exact in every order -> bit-exact wire
    x = oracle.synth(n, 900 + n)
    w = OB.encode(torch.as_tensor(x).cuda()).cpu().numpy()
    assert np.array_equal(w, oracle.onebit_encode_wire(x))
    y = OB.decode(torch.as_tensor(w).cuda(), n).cpu().numpy()
    assert np.array_equal(y.view(np.uint32), oracle.onebit_decode_wire(w, n).view(np.uint32))
    # signed zeros: bit = !signbit, so -0.0 decodes to -scale (kernels.cpp:58-63)
    z = np.array([0.0, -0.0, 1.0, -1.0] * 9, np.float32)
    assert np.array_equal(OB.encode(z), oracle.onebit_encode_wire(z))


def test_onebit_compensate_encode(oracle):
    n = 100_003
    x = oracle.synth(n, 4242)
    d0 = (oracle.synth(n, 4243) * np.float32(0.25)).astype(np.float32)
    d = torch.as_tensor(d0).cuda()
    dec = []
    w = b2.compensate_encode(OB, torch.as_tensor(x).cuda(), d, decoded=dec)
    y = (x - d0).astype(np.float32)
    w_ref = oracle.onebit_encode_wire(y)
    assert np.array_equal(w.cpu().numpy(), w_ref)
    dref = oracle.onebit_decode_wire(w_ref, n)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), (y - dref).astype(np.float32).view(np.uint32))


SIZES = [0, 1, 3, 7, 8, 9, 15, 16, 17, 64, 1000, 4097, 65537, 1_000_003]


@pytest.mark.parametrize("n", SIZES)
def test_random_vs_oracle(oracle, n):
    rng = np.random.default_rng(n + 11)
    x = (rng.standard_normal(n) * 10).astype(np.float32)
    codes, hdr = enc(x)
    if n == 0:
        assert list(hdr) == [0.0, 0.0]
        return
    lo, hi, want = oracle.encode(x)
    assert hdr[0] == lo and hdr[1] == hi
    assert np.array_equal(codes, want)
    got = U8.decode_soa(torch.as_tensor(codes).cuda(), dev(list(hdr) + [0, 0]),
                        torch.empty(n, device="cuda")).cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle.decode(lo, hi, want)))


def test_decode_random_codes(oracle):
    # random codes (every level, not just those a gaussian reaches) at a
    # small and a > 32Mi size, ragged tails: bit-exact vs the oracle
    rng = np.random.default_rng(5)
    for n in (16 * 12345 + 15, (32 << 20) + 17):
        codes = rng.integers(0, 256, n, dtype=np.uint8)
        lo, hi = np.float32(-1.7), np.float32(2.3)
        got = U8.decode_soa(torch.as_tensor(codes).cuda(), dev([lo, hi, 0, 0]),
                            torch.empty(n, device="cuda")).cpu().numpy()
        assert np.array_equal(bits(got), bits(oracle.decode(lo, hi, codes)))


@pytest.mark.parametrize("offset", [1, 2, 3, 5])
def test_unaligned_views(oracle, offset):
    # misaligned device views take the staging path and stay bit-exact
    n = 1031
    base = torch.as_tensor(np.random.default_rng(offset).standard_normal(n + 8).astype(np.float32)).cuda()
    x = base[offset:offset + n]
    codes, hdr = U8.encode_soa(x)
    lo, hi, want = oracle.encode(x.cpu().numpy())
    assert np.array_equal(codes.cpu().numpy(), want)


def test_acceptance_c3_shapes(oracle):
    # acceptance.cpp:197-214: 32-element chunks in [-30, 30); bit-exact vs the
    # oracle and within one step of the input (the north_star tolerance).
    rng = np.random.default_rng(50000)
    for trial in range(300):
        x = rng.uniform(-30, 30, 32).astype(np.float32)
        codes, hdr = enc(x)
        lo, hi, want = oracle.encode(x)
        assert np.array_equal(codes, want) and hdr[0] == lo and hdr[1] == hi
        y = oracle.decode(lo, hi, codes)
        bound = (float(hi) - float(lo)) / 255.0
        assert np.all(np.abs(y.astype(np.float64) - x) <= bound * (1 + 1e-5))


def test_zero_sign_ties(oracle):
    # +-0 ties: header compared with == (test_kernels.cpp:111), codes/decode exact
    x = np.array([0.0, -0.0, 0.0, -0.0, 1.0, -0.0], np.float32)
    codes, hdr = enc(x)
    lo, hi, want = oracle.encode(x)
    assert hdr[0] == lo and hdr[1] == hi and np.array_equal(codes, want)
    allz = np.array([-0.0, 0.0, -0.0], np.float32)
    codes, hdr = enc(allz)
    got = U8.decode_soa(torch.as_tensor(codes).cuda(), dev(list(hdr) + [0, 0]), torch.empty(3, device="cuda"))
    lo, hi, w = oracle.encode(allz)
    assert np.array_equal(bits(got.cpu().numpy()), bits(oracle.decode(lo, hi, w)))


def test_compensate_encode_vs_oracle(oracle):
    # codec.cpp:125-137; test_codec.cpp:230-244 (residual definition bitwise)
    rng = np.random.default_rng(900)
    for n in [1, 33, 1000, 100_003]:
        x = rng.uniform(-5, 5, n).astype(np.float32)
        d0 = rng.uniform(-0.5, 0.5, n).astype(np.float32)
        dd = dev(d0)
        dec = []
        wire = b2.compensate_encode(U8, dev(x), dd, decoded=dec).cpu().numpy()
        d_or = d0.copy()
        lo, hi, codes, decoded = oracle.compensate_encode(x, d_or)
        assert np.array_equal(wire[8:], codes)
        assert wire[:4].view(np.float32)[0] == lo and wire[4:8].view(np.float32)[0] == hi
        assert np.array_equal(bits(dd.cpu().numpy()), bits(d_or))
        assert np.array_equal(bits(dec[0].cpu().numpy()), bits(decoded))


def test_host_inputs_roundtrip(oracle):
    # drop-in path: numpy in, numpy payload out (the reference's Payload)
    x = np.random.default_rng(3).standard_normal(777).astype(np.float32)
    p = U8.encode(x)
    assert isinstance(p, np.ndarray) and p.size == 8 + 777
    assert np.array_equal(p, oracle.encode_wire(x))
    y = U8.decode(p, 777)
    lo, hi, c = oracle.encode(x)
    assert np.array_equal(bits(y), bits(oracle.decode(lo, hi, c)))


def test_golden_fixtures():
    """Reference outputs captured from oracle/_ref (tests/golden/make_golden.py)."""
    path = os.path.join(GOLDEN, "codec_golden.npz")
    if not os.path.exists(path):
        pytest.skip("golden fixtures not generated")
    z = np.load(path)
    for i in range(int(z["count"])):
        x, wire = z[f"x{i}"], z[f"wire{i}"]
        got = U8.encode(dev(x)).cpu().numpy()
        assert np.array_equal(got[8:], wire[8:])
        assert got[:4].view(np.float32)[0] == wire[:4].view(np.float32)[0]
        assert got[4:8].view(np.float32)[0] == wire[4:8].view(np.float32)[0]
        dec = U8.decode(torch.as_tensor(wire).cuda(), x.size).cpu().numpy()
        assert same(dec, z[f"dec{i}"])


# ------------------------------------------------- stochastic rounding
def test_stochastic_rounding_unbiased():
    # test_codec.cpp:175-192, vectorised: one bucket with the reference's three
    # values, the third repeated, every element an independent draw
    import random
    st = b2.Codec(b2.CodecKind.uniform8, b2.Rounding.stochastic)
    draws = 200_000
    x = np.full(draws + 2, 0.3777, np.float32)
    x[0], x[1] = 0.0, 1.0
    rng = random.Random(11)
    w1 = st.encode(dev(x), rng)
    y = st.decode(w1, x.size).cpu().numpy().astype(np.float64)
    assert y[0] == 0.0 and y[1] == 1.0
    e = y[2:] - 0.3777
    assert abs(e.mean()) <= 3.0 * np.sqrt(e.var() / draws)
    codes = w1.cpu().numpy()[8:]
    q = (np.float32(0.3777) - np.float32(0.0)) * np.float32(255.0)
    assert set(np.unique(codes[2:]).tolist()) <= {int(np.floor(q)), int(np.floor(q)) + 1}
    w2 = st.encode(dev(x), rng)  # the generator advanced: different draws
    assert not torch.equal(w1, w2)
    w3 = st.encode(dev(x), random.Random(11))  # same stream: same draws
    assert torch.equal(w1, w3)
    with pytest.raises(b2.Error):
        st.encode(dev([1.0, 2.0]), None)  # codec.cpp:68
