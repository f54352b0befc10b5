"""B200-native rcomm hot path (Bagua communication primitives, arXiv 2107.01499).

Python plumbing over the C ABI of ``libb2comm.so`` (include/b2comm.h); the
compute runs in hand-written sm_100a kernels.  Names mirror the reference's
C++ API (rcomm: collectives.hpp, codec.hpp, tensor.hpp).
"""
from ._lib import B2Error, Error, lib  # noqa: F401  (fails loudly if the .so is missing)
from .codec import Codec, CodecKind, ErrorState, Rounding, compensate_encode  # noqa: F401
from .collectives import (  # noqa: F401
    B200Endpoint,
    ReduceMode,
    ThreadBootstrap,
    Topology,
    TopologyKind,
    TorchBootstrap,
    c_fp_s,
    c_lp_s,
    d_fp_s,
    d_lp_s,
    hierarchical_c,
    owned_partition_len,
    partition_range,
    phase,
)
from .tensor import BucketArena, FlatTensor, TensorView  # noqa: F401
from .engine import OverlapEngine, plan_buckets  # noqa: F401

__all__ = [
    "OverlapEngine", "plan_buckets",
    "B200Endpoint", "BucketArena", "Codec", "CodecKind", "Error", "ErrorState", "FlatTensor", "ReduceMode",
    "Rounding", "TensorView", "ThreadBootstrap", "Topology", "TopologyKind", "TorchBootstrap", "c_fp_s",
    "c_lp_s", "compensate_encode", "d_fp_s", "d_lp_s", "hierarchical_c", "owned_partition_len", "partition_range", "phase",
]
