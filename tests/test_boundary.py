"""The drop-in boundary without a GPU: libb2comm.so loads, exports every
entry point include/b2comm.h declares, carries sm_100a code with the
instructions the design relies on, and its host-only functions agree with
the reference (partition_range, payload_size, Topology::neighbors incl. the
libstdc++-shuffle random matching)."""
import json
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "b2comm.h")
GOLDEN = os.path.join(REPO, "tests", "golden")


@pytest.fixture(scope="module")
def b2lib():
    from paper_2107_01499_b200 import _lib
    return _lib


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(b2_[a-z0-9_]+)\s*\(", txt)) - {"b2_allgather_fn"})


def test_header_symbols_exported(b2lib):
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(b2lib.lib, s), s
    # and the ctypes binding covers exactly the declared surface
    assert sorted(b2lib.EXPORTED) == syms
    out = subprocess.run(["nm", "-D", "--defined-only", b2lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (b2_\w+)", out))
    assert set(syms) == exported, set(syms) ^ exported


def test_no_cpu_fallback_without_gpu(b2lib):
    """Without a device the library refuses to create a communicator (and the
    codec launches fail) instead of silently computing on the CPU."""
    import ctypes as C
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    h = C.c_void_p()
    cb = b2lib.ALLGATHER_FN(lambda *a: 1)
    assert b2lib.lib.b2_comm_create(1, 0, 0, cb, None, C.byref(h)) != b2lib.B2_OK
    x = (C.c_float * 64)()
    hdr = (C.c_float * 4)()
    codes = (C.c_uint8 * 64)()
    rc = b2lib.lib.b2_u8_encode(C.addressof(x), 64, C.addressof(codes), C.addressof(hdr), None)
    assert rc == b2lib.B2_ERR_CUDA


def test_sm100a_sass_and_tma(b2lib):
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    listing = subprocess.run([cuobjdump, "--list-elf", b2lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in listing
    sass = subprocess.run([cuobjdump, "-sass", b2lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # cp.async.bulk (TMA) ring
    assert "SYNCS.PHASECHK" in sass  # mbarrier waits
    assert "REDUX" in sass or "CREDUX" in sass  # redux.sync min/max


def test_partition_range_and_payload(b2lib):
    import paper_2107_01499_b200 as b2
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        k = json.load(f)
    for n, g, i, lo, sz in k["partition_range"]["cases"]:
        assert b2.partition_range(n, g, i) == (lo, sz)
    for n, w, i, own in k["partition_range"]["owned"]:
        assert b2.owned_partition_len(n, w, i) == own
    p = k["payload_size"]
    assert b2.Codec(b2.CodecKind.identity).payload_size(4) == p["identity_4"]
    assert b2.Codec(b2.CodecKind.uniform8).payload_size(4) == p["uniform8_4"]
    assert b2.Codec(b2.CodecKind.onebit).payload_size(9) == p["onebit_9"]
    # tiling property: partitions cover [0, len) in order, sizes differ by <= 1
    for n in (0, 1, 7, 1000, 100_000_007):
        for g in (1, 2, 3, 8):
            parts = [b2.partition_range(n, g, r) for r in range(g)]
            assert parts[0][0] == 0 and sum(s for _, s in parts) == n
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(g - 1))
            assert max(s for _, s in parts) - min(s for _, s in parts) <= 1


def test_topology_matches_reference_golden(b2lib):
    import paper_2107_01499_b200 as b2
    with open(os.path.join(GOLDEN, "topology_golden.json")) as f:
        t = json.load(f)
    for key, want in t["random"].items():
        n, seed, rnd, r = map(int, key.split(","))
        assert b2.Topology(b2.TopologyKind.random, n, seed).neighbors(r, rnd) == want, key
    for key, want in t["ring"].items():
        n, r = map(int, key.split(","))
        assert b2.Topology(b2.TopologyKind.ring, n, 0).neighbors(r, 0) == want
    for key, want in t["full"].items():
        n, r = map(int, key.split(","))
        assert b2.Topology(b2.TopologyKind.full, n, 0).neighbors(r, 0) == want
    with pytest.raises(b2.Error):
        b2.Topology(b2.TopologyKind.ring, 4, 0).neighbors(4, 0)


def test_random_topology_is_a_symmetric_matching():
    # test_collectives.cpp:194-206
    import paper_2107_01499_b200 as b2
    topo = b2.Topology(b2.TopologyKind.random, 8, 123)
    for rnd in range(20):
        for r in range(8):
            nb = topo.neighbors(r, rnd)
            assert len(nb) == 2 and r in nb
            for p in nb:
                assert r in topo.neighbors(p, rnd)


def test_codec_host_errors():
    import paper_2107_01499_b200 as b2
    with pytest.raises(b2.Error, match="needs a generator"):
        b2.Codec(b2.CodecKind.uniform8, b2.Rounding.stochastic)._check_supported(None)
    import random
    c = b2.Codec(b2.CodecKind.uniform8, b2.Rounding.stochastic)
    c._check_supported(random.Random(1))  # the collectives take stochastic rounding (b2_c_lp_s_stochastic)
    c._check_supported(random.Random(1), collective=False)
    assert c.stochastic() and not b2.Codec(b2.CodecKind.uniform8).stochastic()
    r = random.Random(5)
    s1 = c._seed(r)
    assert s1 != c._seed(r)  # the generator advances per call (codec.cpp:71-74)
    b2.Codec(b2.CodecKind.onebit)._check_supported(None)  # every primitive takes the onebit codec
    assert b2.phase.make_tag(3, b2.phase.bcast) == 51


def test_status_strings(b2lib):
    assert b2lib.lib.b2_status_string(b2lib.B2_ERR_NONFINITE) == b"encode: non-finite input value"
    assert b2lib.lib.b2_version() == 1


def test_hierarchical_node_groups():
    # collectives.cpp:299-310: members ascending per node, leaders = lowest member, ascending
    from paper_2107_01499_b200.collectives import _node_groups
    assert _node_groups([0, 0, 0, 1, 1, 2]) == ([[0, 1, 2], [3, 4], [5]], [0, 3, 5])
    assert _node_groups([2, 0, 1, 0, 2, 1]) == ([[1, 3], [2, 5], [0, 4]], [0, 1, 2])
