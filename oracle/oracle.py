"""ctypes bindings for the C restatement and the compiled reference (test infra)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
_REF_SRC = "/root/reference/proj"

_f32p = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)
_sz = C.c_size_t


def build(force: bool = False) -> None:
    """Build liboracle.so (always) and _ref/librcomm_ref.so (only where the
    reference tree exists, i.e. in the authoring container)."""
    targets = ["oracle"]
    if os.path.isdir(_REF_SRC):
        targets.append("ref")
    cmd = ["make", "-C", ORACLE_DIR] + (["-B"] if force else []) + targets
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)


def _f(a: np.ndarray):
    return a.ctypes.data_as(_f32p)


def _ptr_array(arrs):
    return (_f32p * len(arrs))(*[_f(a) for a in arrs])


class Oracle:
    """The plain-C restatement (rcomm_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(ORACLE_DIR, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_partition_range.argtypes = [_sz, C.c_int, C.c_int, C.POINTER(_sz), C.POINTER(_sz)]
        L.orc_minmax.argtypes = [_f32p, _sz, _f32p, _f32p]
        L.orc_quantize_u8.argtypes = [_f32p, _u8p, C.c_float, C.c_float, _sz]
        L.orc_u8_encode.argtypes = [_f32p, _sz, _f32p, _f32p, _u8p]
        L.orc_u8_decode.argtypes = [C.c_float, C.c_float, _u8p, _sz, _f32p]
        L.orc_u8_encode_wire.argtypes = [_f32p, _sz, _u8p]
        L.orc_onebit_encode_wire.argtypes = [_f32p, _sz, _u8p]
        L.orc_onebit_decode_wire.argtypes = [_u8p, _sz, _f32p]
        L.orc_u8_compensate_encode.argtypes = [_f32p, _f32p, _sz, _f32p, _f32p, _u8p, _f32p]
        L.orc_c_fp_s.argtypes = [C.c_int, _sz, C.POINTER(_f32p)]
        L.orc_c_lp_s.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.c_int, C.POINTER(_f32p), C.POINTER(_f32p)]
        L.orc_hierarchical_c.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.POINTER(C.c_int), C.c_int]
        L.orc_d_fp_s_rank.argtypes = [_sz, C.POINTER(_f32p), C.c_int, C.c_int, _f32p]
        L.orc_d_lp_s_rank.argtypes = [_sz, C.POINTER(_f32p), C.c_int, C.c_int, C.c_int, _f32p]
        L.orc_topology_neighbors.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.orc_synth.argtypes = [_f32p, _sz, C.c_uint64, C.c_uint64]

    def partition_range(self, length: int, n: int, k: int):
        lo, sz = _sz(), _sz()
        self.lib.orc_partition_range(length, n, k, C.byref(lo), C.byref(sz))
        return lo.value, sz.value

    def minmax(self, x):
        x = np.ascontiguousarray(x, np.float32)
        lo, hi = C.c_float(), C.c_float()
        self.lib.orc_minmax(_f(x), x.size, C.byref(lo), C.byref(hi))
        return np.float32(lo.value), np.float32(hi.value)

    def quantize_u8(self, x, mn, inv_step):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(x.size, np.uint8)
        self.lib.orc_quantize_u8(_f(x), out.ctypes.data_as(_u8p), mn, inv_step, x.size)
        return out

    def encode(self, x):
        """-> (lo, hi, codes) or raises ValueError on non-finite input."""
        x = np.ascontiguousarray(x, np.float32)
        codes = np.zeros(max(x.size, 1), np.uint8)
        lo, hi = C.c_float(), C.c_float()
        rc = self.lib.orc_u8_encode(_f(x), x.size, C.byref(lo), C.byref(hi), codes.ctypes.data_as(_u8p))
        if rc:
            raise ValueError("encode: non-finite input value")
        return np.float32(lo.value), np.float32(hi.value), codes[: x.size]

    def decode(self, lo, hi, codes):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.zeros(codes.size, np.float32)
        self.lib.orc_u8_decode(lo, hi, codes.ctypes.data_as(_u8p), codes.size, _f(out))
        return out

    def encode_wire(self, x):
        x = np.ascontiguousarray(x, np.float32)
        wire = np.zeros(8 + x.size, np.uint8)
        if self.lib.orc_u8_encode_wire(_f(x), x.size, wire.ctypes.data_as(_u8p)):
            raise ValueError("encode: non-finite input value")
        return wire

    def onebit_encode_wire(self, x):
        """codec.cpp:81-88 (scalar kernels): [scale f32][ceil(n/8) sign bytes]."""
        x = np.ascontiguousarray(x, np.float32)
        wire = np.zeros(4 + (x.size + 7) // 8, np.uint8)
        if self.lib.orc_onebit_encode_wire(_f(x), x.size, wire.ctypes.data_as(_u8p)):
            raise ValueError("encode: non-finite input value")
        return wire

    def onebit_decode_wire(self, wire, n):
        wire = np.ascontiguousarray(wire, np.uint8)
        out = np.zeros(max(n, 1), np.float32)
        self.lib.orc_onebit_decode_wire(wire.ctypes.data_as(_u8p), n, _f(out))
        return out[:n]

    def compensate_encode(self, x, delta):
        """delta is updated in place; returns (lo, hi, codes, decoded)."""
        x = np.ascontiguousarray(x, np.float32)
        assert delta.dtype == np.float32 and delta.flags.c_contiguous
        codes = np.zeros(max(x.size, 1), np.uint8)
        dec = np.zeros(max(x.size, 1), np.float32)
        lo, hi = C.c_float(), C.c_float()
        rc = self.lib.orc_u8_compensate_encode(_f(x), _f(delta), x.size, C.byref(lo), C.byref(hi),
                                               codes.ctypes.data_as(_u8p), _f(dec))
        if rc:
            raise ValueError("encode: non-finite input value")
        return np.float32(lo.value), np.float32(hi.value), codes[: x.size], dec[: x.size]

    def c_fp_s(self, xs):
        """xs: list of g float32 arrays, updated in place."""
        self.lib.orc_c_fp_s(len(xs), xs[0].size, _ptr_array(xs))

    def c_lp_s(self, xs, codec=1, deltas=None, eps=None):
        rc = self.lib.orc_c_lp_s(len(xs), xs[0].size, _ptr_array(xs), codec,
                                 _ptr_array(deltas) if deltas is not None else None,
                                 _ptr_array(eps) if eps is not None else None)
        if rc:
            raise ValueError("encode: non-finite input value")

    def hierarchical_c(self, xs, nodes, codec=1):
        arr = (C.c_int * len(nodes))(*nodes)
        rc = self.lib.orc_hierarchical_c(len(xs), xs[0].size, _ptr_array(xs), arr, codec)
        if rc:
            raise ValueError("encode: non-finite input value")

    def d_fp_s_rank(self, nbr_xs, mode=1):
        out = np.zeros(nbr_xs[0].size, np.float32)
        self.lib.orc_d_fp_s_rank(out.size, _ptr_array(nbr_xs), len(nbr_xs), mode, _f(out))
        return out

    def d_lp_s_rank(self, nbr_xs, codec=1, mode=1):
        out = np.zeros(nbr_xs[0].size, np.float32)
        rc = self.lib.orc_d_lp_s_rank(out.size, _ptr_array(nbr_xs), len(nbr_xs), codec, mode, _f(out))
        if rc:
            raise ValueError("encode: non-finite input value")
        return out

    def neighbors(self, kind_ring1_full2: int, n: int, rank: int):
        out = (C.c_int * max(n, 3))()
        m = self.lib.orc_topology_neighbors(kind_ring1_full2, n, rank, out)
        if m < 0:
            raise ValueError("topology: rank out of range")
        return list(out[:m])

    def synth(self, n: int, seed: int, offset: int = 0):
        out = np.empty(n, np.float32)
        self.lib.orc_synth(_f(out), n, seed, offset)
        return out


class Reference:
    """The unmodified reference library (oracle/_ref/librcomm_ref.so)."""

    PATH = os.path.join(ORACLE_DIR, "_ref", "librcomm_ref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        if not self.available():
            build()
        L = self.lib = C.CDLL(self.PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_backend.restype = C.c_char_p
        L.ref_encode.argtypes = [C.c_int, _f32p, _sz, _u8p]
        L.ref_decode.argtypes = [C.c_int, _u8p, _sz, _sz, _f32p]
        L.ref_compensate_encode.argtypes = [C.c_int, _f32p, _f32p, _sz, _u8p, _f32p]
        L.ref_quantize_u8.argtypes = [_f32p, _u8p, C.c_float, C.c_float, _sz]
        L.ref_minmax.argtypes = [_f32p, _sz, _f32p, _f32p]
        L.ref_c_fp_s.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.ref_c_lp_s.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.c_int, C.POINTER(_f32p),
                                 C.POINTER(_f32p), C.c_int, C.POINTER(C.c_uint64)]
        L.ref_hierarchical_c.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.POINTER(C.c_int), C.c_int]
        L.ref_d_fp_s.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.c_int, C.c_uint64, C.c_uint64, C.c_int]
        L.ref_d_lp_s.argtypes = [C.c_int, _sz, C.POINTER(_f32p), C.c_int, C.c_uint64, C.c_uint64,
                                 C.c_int, C.c_int]
        L.ref_neighbors.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_int)]
        L.ref_random_uniform.argtypes = [C.c_uint32, _sz, C.c_float, C.c_float, _f32p]
        L.ref_random_normal.argtypes = [C.c_uint32, _sz, _f32p]
        L.ref_synth.argtypes = [_f32p, _sz, C.c_uint64]
        L.ref_time_primitive.argtypes = [C.c_int, C.c_int, _sz, C.c_int, C.POINTER(C.c_double)]
        L.ref_force_backend.argtypes = [C.c_int]

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def backend(self) -> str:
        return self.lib.ref_backend().decode()

    def encode(self, x, codec=1):
        x = np.ascontiguousarray(x, np.float32)
        size = {0: 4 * x.size, 1: 8 + x.size, 2: 4 + (x.size + 7) // 8}[codec]
        wire = np.zeros(size + 1, np.uint8)
        self._check(self.lib.ref_encode(codec, _f(x), x.size, wire.ctypes.data_as(_u8p)))
        return wire[:size]

    def decode(self, wire, n, codec=1):
        wire = np.ascontiguousarray(wire, np.uint8)
        out = np.zeros(max(n, 1), np.float32)
        self._check(self.lib.ref_decode(codec, wire.ctypes.data_as(_u8p), wire.size, n, _f(out)))
        return out[:n]

    def compensate_encode(self, x, delta, codec=1):
        x = np.ascontiguousarray(x, np.float32)
        wire = np.zeros(8 + x.size, np.uint8)
        dec = np.zeros(max(x.size, 1), np.float32)
        self._check(self.lib.ref_compensate_encode(codec, _f(x), _f(delta), x.size,
                                                   wire.ctypes.data_as(_u8p), _f(dec)))
        return wire, dec[: x.size]

    def quantize_u8(self, x, mn, inv_step):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(max(x.size, 1), np.uint8)
        self.lib.ref_quantize_u8(_f(x), out.ctypes.data_as(_u8p), mn, inv_step, x.size)
        return out[: x.size]

    def minmax(self, x):
        x = np.ascontiguousarray(x, np.float32)
        lo, hi = C.c_float(), C.c_float()
        self.lib.ref_minmax(_f(x), x.size, C.byref(lo), C.byref(hi))
        return np.float32(lo.value), np.float32(hi.value)

    def c_fp_s(self, xs):
        g = len(xs)
        b = (C.c_uint64 * g)()
        m = (C.c_uint64 * g)()
        self._check(self.lib.ref_c_fp_s(g, xs[0].size, _ptr_array(xs), b, m))
        return list(b), list(m)

    def c_lp_s(self, xs, codec=1, deltas=None, eps=None, rounds=1):
        g = len(xs)
        b = (C.c_uint64 * g)()
        self._check(self.lib.ref_c_lp_s(g, xs[0].size, _ptr_array(xs), codec,
                                        _ptr_array(deltas) if deltas is not None else None,
                                        _ptr_array(eps) if eps is not None else None, rounds, b))
        return list(b)

    def hierarchical_c(self, xs, nodes, codec=1):
        arr = (C.c_int * len(nodes))(*nodes)
        self._check(self.lib.ref_hierarchical_c(len(xs), xs[0].size, _ptr_array(xs), arr, codec))

    def d_fp_s(self, xs, topo_kind=0, seed=0, round_=0, mode=1):
        self._check(self.lib.ref_d_fp_s(len(xs), xs[0].size, _ptr_array(xs), topo_kind, seed, round_, mode))

    def d_lp_s(self, xs, topo_kind=0, seed=0, round_=0, codec=1, mode=1):
        self._check(self.lib.ref_d_lp_s(len(xs), xs[0].size, _ptr_array(xs), topo_kind, seed, round_,
                                        codec, mode))

    def neighbors(self, topo_kind: int, n: int, seed: int, rank: int, round_: int):
        out = (C.c_int * max(n, 3))()
        m = self.lib.ref_neighbors(topo_kind, n, seed, rank, round_, out)
        if m < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return list(out[:m])

    def random_uniform(self, seed, n, lo, hi):
        out = np.zeros(max(n, 1), np.float32)
        self.lib.ref_random_uniform(seed, n, lo, hi, _f(out))
        return out[:n]

    def random_normal(self, seed, n):
        out = np.zeros(max(n, 1), np.float32)
        self.lib.ref_random_normal(seed, n, _f(out))
        return out[:n]

    def synth(self, n, seed):
        out = np.empty(n, np.float32)
        self.lib.ref_synth(_f(out), n, seed)
        return out

    def time_primitive(self, prim: int, g: int, n: int, reps: int):
        secs = (C.c_double * reps)()
        self._check(self.lib.ref_time_primitive(prim, g, n, reps, secs))
        return list(secs)
