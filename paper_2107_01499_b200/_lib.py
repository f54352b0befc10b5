"""ctypes binding of libb2comm.so (include/b2comm.h).

The product path: every compute call below lands in the in-tree CUDA library.
There is no CPU fallback -- if the library is missing, import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# B2COMM_LIB: an alternative in-tree build of the same library (A/B runs of
# compile-time variants, paper_2107_01499_b200/build.py build_variant)
LIB_PATH = os.environ.get("B2COMM_LIB") or os.path.join(PKG_DIR, "libb2comm.so")

B2_OK, B2_ERR_INVALID, B2_ERR_CUDA, B2_ERR_NONFINITE, B2_ERR_TIMEOUT, B2_ERR_UNSUPPORTED, B2_ERR_BOOTSTRAP = range(7)
CODEC_IDENTITY, CODEC_UNIFORM8, CODEC_ONEBIT = 0, 1, 2
REDUCE_SUM, REDUCE_AVERAGE = 0, 1
TOPO_RING, TOPO_RANDOM, TOPO_FULL = 0, 1, 2
MAX_RANKS = 8
U8_HDR_BYTES = 16

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

# name -> (restype, argtypes); the exported surface of include/b2comm.h
_SIGS = {
    "b2_version": (C.c_int, []),
    "b2_last_error": (C.c_char_p, []),
    "b2_status_string": (C.c_char_p, [C.c_int]),
    "b2_partition_range": (None, [C.c_size_t, C.c_int, C.c_int, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "b2_owned_partition_len": (C.c_size_t, [C.c_size_t, C.c_int, C.c_int]),
    "b2_payload_size": (C.c_size_t, [C.c_int, C.c_size_t]),
    "b2_topology_neighbors": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.POINTER(C.c_int)]),
    "b2_u8_encode": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2_u8_encode_stochastic": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "b2_u8_decode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "b2_u8_compensate_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]),
    "b2_u8_pack_wire": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "b2_identity_compensate_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                                C.c_void_p]),
    "b2_onebit_compensate_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                              C.c_void_p]),
    "b2_onebit_encode": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "b2_onebit_decode": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "b2_u8_unpack_wire": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p]),
    "b2_bucket_flatten": (C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int, C.c_void_p, C.c_void_p]),
    "b2_bucket_unflatten": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int, C.c_void_p]),
    "b2_fill_synthetic": (C.c_int, [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64, C.c_void_p]),
    "b2_comm_create": (C.c_int, [C.c_int, C.c_int, C.c_int, ALLGATHER_FN, C.c_void_p, C.POINTER(C.c_void_p)]),
    "b2_comm_destroy": (C.c_int, [C.c_void_p]),
    "b2_comm_rank": (C.c_int, [C.c_void_p]),
    "b2_comm_world": (C.c_int, [C.c_void_p]),
    "b2_comm_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "b2_comm_poll": (C.c_int, [C.c_void_p]),
    "b2_comm_set_timeout_ms": (C.c_int, [C.c_void_p, C.c_uint64]),
    "b2_comm_launches": (C.c_uint64, [C.c_void_p]),
    "b2_comm_poisoned": (C.c_int, [C.c_void_p]),
    "b2_comm_set_sm_budget": (C.c_int, [C.c_void_p, C.c_int]),
    "b2_comm_release_bucket": (C.c_int, [C.c_void_p, C.c_uint32]),
    "b2_comm_window_bytes": (C.c_size_t, [C.c_void_p]),
    "b2_comm_enable_trace": (C.c_int, [C.c_void_p, C.c_int]),
    "b2_comm_read_trace": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_int)]),
    "b2_c_fp_s": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32, C.c_void_p]),
    "b2_c_lp_s": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_size_t,
                            C.c_void_p, C.c_size_t, C.c_uint32, C.c_void_p]),
    "b2_hierarchical_c": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32, C.c_void_p]),
    "b2_c_lp_s_stochastic": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_void_p,
                                       C.c_size_t, C.c_uint64, C.c_uint32, C.c_void_p]),
    "b2_d_lp_s_stochastic": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_int), C.c_int, C.c_int,
                                       C.c_uint64, C.c_uint32, C.c_void_p]),
    "b2_d_fp_s": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_int), C.c_int, C.c_int,
                            C.c_uint32, C.c_void_p]),
    "b2_d_lp_s": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_int), C.c_int, C.c_int,
                            C.c_int, C.c_uint32, C.c_void_p]),
}

EXPORTED = tuple(_SIGS)


class Error(RuntimeError):
    """Mirror of rcomm::Error (tensor.hpp:12-14): every failure the reference
    reports by throwing surfaces as this exception."""


class B2Error(Error):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 hot path)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    return (lib.b2_last_error() or b"").decode()


def check(status: int) -> None:
    if status != B2_OK:
        raise B2Error(status, f"{lib.b2_status_string(status).decode()}: {last_error()}")
