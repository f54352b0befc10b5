"""The four synchronous primitives behind rcomm's API (collectives.hpp:13-89).

``B200Endpoint`` stands where rcomm's ``Endpoint`` stands (transport.hpp:52-85):
one per worker (process or thread), bound to one GPU.  The primitive
functions keep the reference signatures -- ``c_lp_s(ep, now, x, codec, es,
rng=None, bucket=0)`` etc. -- update ``x`` in place, are blocking by default
(the reference's rendezvous semantics) and return ``now`` unchanged (there is
no virtual clock on real hardware; TcpEndpoint likewise passes clocks
through, transport.hpp:276-279).

``x`` may be a CUDA float32 tensor (zero-copy), a FlatTensor / BucketArena,
or a host buffer (numpy array / CPU tensor), which is staged through pinned
memory -- the end-to-end path a drop-in user of host vectors gets.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import enum
import os
import threading

import numpy as np
import torch

from . import _lib
from ._lib import Error, check, lib
from .codec import Codec, CodecKind, ErrorState, Rounding


class TopologyKind(enum.IntEnum):
    ring = _lib.TOPO_RING
    random = _lib.TOPO_RANDOM
    full = _lib.TOPO_FULL


class ReduceMode(enum.IntEnum):
    sum = _lib.REDUCE_SUM
    average = _lib.REDUCE_AVERAGE


class phase:  # collectives.hpp:29-38
    scatter, gather, inter, bcast = 0, 1, 2, 3

    @staticmethod
    def make_tag(bucket: int, ph: int) -> int:
        return bucket * 16 + ph


def partition_range(length: int, n: int, k: int):
    lo, sz = C.c_size_t(), C.c_size_t()
    lib.b2_partition_range(length, n, k, C.byref(lo), C.byref(sz))
    return lo.value, sz.value


def owned_partition_len(length: int, world: int, idx: int) -> int:
    return int(lib.b2_owned_partition_len(length, world, idx))


class Topology:
    """Neighbour function N(i), sorted and self-inclusive (collectives.hpp:18-25)."""

    def __init__(self, kind: TopologyKind = TopologyKind.full, n: int = 1, seed: int = 0):
        self.kind, self.n, self.seed = TopologyKind(kind), int(n), int(seed)

    def neighbors(self, rank: int, round_: int) -> list[int]:
        return list(self._neighbors_c(rank, round_)[0])

    def _neighbors_c(self, rank: int, round_: int):
        """-> (ctypes int array, count); ring / full do not depend on the round
        and are cached (the per-call host cost matters for small buckets)."""
        key = (int(self.kind), self.n, self.seed, rank, 0 if self.kind != TopologyKind.random else round_)
        hit = _NBR_CACHE.get(key)
        if hit is not None:
            return hit
        out = (C.c_int * max(self.n, 3))()
        m = lib.b2_topology_neighbors(int(self.kind), self.n, self.seed & (2**64 - 1), rank,
                                      int(round_) & (2**64 - 1), out)
        if m < 0:
            raise Error(_lib.last_error())
        res = ((C.c_int * m)(*out[:m]), m)
        if self.kind != TopologyKind.random:
            _NBR_CACHE[key] = res
        return res


_NBR_CACHE: dict = {}


# --------------------------------------------------------------- bootstrap
class TorchBootstrap:
    """Window-handle exchange over a gloo group of torch.distributed."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group if group is not None else dist.new_group(backend="gloo")

    def allgather(self, data: bytes, world: int) -> list[bytes]:
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        outs = [torch.empty_like(t) for _ in range(world)]
        self.dist.all_gather(outs, t, group=self.group)
        return [o.numpy().tobytes() for o in outs]


class ThreadBootstrap:
    """In-process exchange for one thread per GPU (SimCluster's threading
    model, sim_transport.cpp:93-128).  Share one instance among the threads."""

    def __init__(self, world: int):
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots: list[bytes | None] = [None] * world
        self._rank = threading.local()

    def allgather(self, data: bytes, world: int, rank: int) -> list[bytes]:
        self._slots[rank] = data
        self._barrier.wait()
        out = list(self._slots)
        self._barrier.wait()
        return out


class B200Endpoint:
    """One worker's handle on the B200 communicator (libb2comm b2_comm_t)."""

    def __init__(self, rank: int | None = None, world_size: int | None = None, device: int | None = None,
                 bootstrap=None, timeout_ms: int | None = None):
        import torch.distributed as dist
        if rank is None or world_size is None:
            if dist.is_available() and dist.is_initialized():
                rank, world_size = dist.get_rank(), dist.get_world_size()
            else:
                rank, world_size = 0, 1
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank)) % max(torch.cuda.device_count(), 1)
        self._rank, self._world, self.device = int(rank), int(world_size), int(device)
        if bootstrap is None and self._world > 1:
            bootstrap = TorchBootstrap()
        self._bootstrap = bootstrap
        self._cb = _lib.ALLGATHER_FN(self._allgather)  # keep alive
        self._bytes_sent = 0
        self._acct: dict = {}  # per-(primitive, codec, n) bytes sent, cached
        self._messages_sent = 0
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(lib.b2_comm_create(self._world, self._rank, self.device, self._cb, None, C.byref(h)))
        self._h = h
        if timeout_ms is not None:  # default: the library's (b2comm.h, 10 min)
            check(lib.b2_comm_set_timeout_ms(h, int(timeout_ms)))

    def _allgather(self, user, send, nbytes, recv) -> int:
        try:
            data = C.string_at(send, nbytes)
            if isinstance(self._bootstrap, ThreadBootstrap):
                parts = self._bootstrap.allgather(data, self._world, self._rank)
            else:
                parts = self._bootstrap.allgather(data, self._world)
            blob = b"".join(parts)
            C.memmove(recv, blob, len(blob))
            return 0
        except Exception:  # surfaced to C as B2_ERR_BOOTSTRAP
            return 1

    # Endpoint interface (transport.hpp:214-242)
    def rank(self) -> int:
        return self._rank

    def world_size(self) -> int:
        return self._world

    def node(self) -> int:
        return 0

    def node_of(self, rank: int) -> int:
        if not 0 <= rank < self._world:
            raise Error(f"unknown rank {rank}")
        return 0

    def bytes_sent(self) -> int:
        return self._bytes_sent

    def messages_sent(self) -> int:
        return self._messages_sent

    def reset_counters(self) -> None:
        self._bytes_sent = self._messages_sent = 0

    def launches(self) -> int:
        return int(lib.b2_comm_launches(self._h))

    def set_sm_budget(self, sms: int) -> None:
        """Launch every primitive on `sms` SMs (0: all), leaving the others to
        concurrent compute.  Every rank must set the same budget (b2comm.h)."""
        check(lib.b2_comm_set_sm_budget(self._h, int(sms)))

    def poll(self) -> None:
        """Raise a latched device error (non-finite input, timeout) without
        synchronizing."""
        check(lib.b2_comm_poll(self._h))

    def poisoned(self) -> bool:
        """True once a rendezvous timed out: every further primitive raises
        until the endpoint is closed and re-created (b2comm.h)."""
        return bool(lib.b2_comm_poisoned(self._h))

    def release_bucket(self, bucket: int) -> None:
        """Collective: free every peer window of `bucket` (b2_comm_release_bucket)."""
        check(lib.b2_comm_release_bucket(self._h, int(bucket)))

    def window_bytes(self) -> int:
        return int(lib.b2_comm_window_bytes(self._h))

    # -- phase tracing (ncu cannot replay kernels that rendezvous across GPUs)
    TRACE_POINTS = ("start", "p1_first_minmax", "p1_first_push", "p1_done", "p2_ready", "p2_minmax",
                    "p2_done", "p3_first", "end", "p2_pass") + tuple(f"p1_step{i}" for i in range(8)) + tuple(
                    f"p1_fenced{i}" for i in range(8))
    # accumulated waits (ns -> us, not timestamps) of the traced stream:
    # (C_LP_S phase 1B) encode consumers on a free credit, fold producer on
    # arrival gates, encode producer on a free stage, signaller in fences,
    # encode / fold consumers on a full stage
    WAIT_POINTS = ("w_slot", "w_gate", "w_empty", "w_retire", "w_full", "w_fullB")

    def enable_trace(self, on: bool = True) -> None:
        check(lib.b2_comm_enable_trace(self._h, int(on)))

    def read_trace(self, raw: bool = False):
        """-> {point: (median, max) microseconds after the earliest CTA start}
        for the last primitive launched (synchronizes the device); raw=True
        returns the [CTA, point] array in microseconds instead."""
        import numpy as _np
        torch.cuda.synchronize(self.device)
        grid = torch.cuda.get_device_properties(self.device).multi_processor_count
        buf = (C.c_uint64 * (grid * 32))()
        n = C.c_int()
        check(lib.b2_comm_read_trace(self._h, buf, grid, C.byref(n)))
        t = _np.ctypeslib.as_array(buf).reshape(grid, n.value).astype(_np.float64)
        t0 = t[:, 0].min()
        if raw:
            return _np.where(t > 0, (t - t0) / 1e3, _np.nan)
        out = {"t0_ns": int(t0)}  # absolute %globaltimer of this rank's first CTA start
        for i, name in enumerate(self.WAIT_POINTS):
            col = t[:, 26 + i]
            col = col[col > 0]
            if col.size:
                out[name] = (round(float(_np.median(col)) / 1e3, 2), round(float(col.max()) / 1e3, 2))
        for i, name in enumerate(self.TRACE_POINTS):
            col = t[:, i]
            col = col[col > 0]
            if col.size:
                out[name] = (round(float(_np.median(col) - t0) / 1e3, 2), round(float(col.max() - t0) / 1e3, 2))
        return out

    @property
    def handle(self):
        return self._h

    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _staging(self) -> "_HostStaging":
        st = self.__dict__.get("_stage")
        if st is None:
            st = self._stage = _HostStaging(self.device)
        return st

    def join(self, stream=None) -> None:
        """Make `stream` (default: current) wait for this endpoint's pending
        host uploads / downloads (non-blocking host buckets)."""
        st = self.__dict__.get("_stage")
        if st is not None:
            st.join(stream or torch.cuda.current_stream(self.device))

    def sync(self) -> None:
        """Wait for this rank's queued primitives (and host copies); raise on
        latched errors."""
        st = self.__dict__.get("_stage")
        if st is not None and st.pending:
            st.join(torch.cuda.current_stream(self.device))
        check(lib.b2_comm_sync(self._h, self.stream()))
        if st is not None:
            st.host_ev.clear()  # every download has landed

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.b2_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _account(self, nbytes: int, msgs: int) -> None:
        self._bytes_sent += nbytes
        self._messages_sent += msgs


# ------------------------------------------------------------ bucket staging
class _HostStaging:
    """Per-endpoint staging of HOST buckets (the drop-in path for callers
    holding gradients in host memory, like the reference's std::vector
    buckets): device buffers are cached per bucket length (a ring of two, so
    the upload of one call overlaps the download of the previous one), pinned
    bounce buffers are cached for pageable inputs, and uploads / downloads run
    on their own streams -- PCIe is full duplex.  Nothing is allocated or
    pinned per call once a length has been seen."""

    RING = 2

    def __init__(self, device: int):
        self.device = device
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self._dev: dict = {}      # n -> [[tensor, free event | None], ...]
        self._next: dict = {}     # n -> next ring slot
        self._bounce: dict = {}   # n -> pinned host tensor
        self.host_ev: dict = {}   # host address -> event of the last download into it
        self.pending = False      # downloads issued since the last join

    def slot(self, n: int):
        ring = self._dev.get(n)
        if ring is None:
            ring = self._dev[n] = [[torch.empty(max(n, 4), dtype=torch.float32,
                                                device=torch.device("cuda", self.device))[:n], None]
                                   for _ in range(self.RING)]
            self._next[n] = 0
        i = self._next[n]
        self._next[n] = (i + 1) % self.RING
        return ring[i]

    def bounce(self, n: int) -> torch.Tensor:
        b = self._bounce.get(n)
        if b is None:
            b = self._bounce[n] = torch.empty(max(n, 4), dtype=torch.float32).pin_memory()[:n]
        return b

    def join(self, stream) -> None:
        """`stream` waits for every upload and download issued so far."""
        stream.wait_stream(self.h2d)
        stream.wait_stream(self.d2h)
        self.pending = False


class _Bucket:
    """Resolve x to an aligned contiguous device float32 tensor.

    Device tensors are used in place.  Host buckets go through the
    endpoint's _HostStaging: a pinned torch tensor is uploaded straight from
    its memory and the result downloaded straight back into it (with
    blocking=False both copies are asynchronous and the result is valid after
    ep.sync()); pageable inputs (numpy, unpinned tensors) go through a cached
    pinned bounce buffer and are always blocking.  The latched device status
    is checked BEFORE a blocking call writes anything back, so a failing call
    (non-finite input, timeout) leaves a host x untouched, as the reference
    throws from encode before x changes (codec.cpp:24-27)."""

    def __init__(self, ep: B200Endpoint, x):
        if (type(x) is torch.Tensor and x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
                and x.data_ptr() % 16 == 0):  # the common case, no staging
            self.orig = self.view = self.dev = x
            self.host = False
            self.n = x.numel()
            return
        from .tensor import BucketArena, FlatTensor
        self.orig = x
        if isinstance(x, (FlatTensor, BucketArena)):
            x = x.data()
        self.host = not (isinstance(x, torch.Tensor) and x.is_cuda)
        self.ep = ep
        if self.host:
            if isinstance(x, torch.Tensor):
                if x.dtype != torch.float32:
                    raise Error("bucket must be float32")
                self.host_t = x
                flat = x.reshape(-1) if x.is_contiguous() else None
            else:
                self.host_t = x
                arr = np.asarray(x)
                if arr.dtype != np.float32:
                    raise Error("bucket must be float32")
                flat = torch.from_numpy(arr).reshape(-1) if arr.flags.c_contiguous else None
            self.n = int(np.prod(np.shape(x))) if not isinstance(x, torch.Tensor) else x.numel()
            st = ep._staging()
            self.pinned = flat is not None and isinstance(x, torch.Tensor) and flat.is_pinned()
            self.src = flat if self.pinned else st.bounce(self.n)
            if not self.pinned:
                self.src.copy_(torch.as_tensor(np.ascontiguousarray(x, np.float32)).reshape(-1)
                               if flat is None else flat)
            self.slot = st.slot(self.n)
            self.dev = self.slot[0]
            with torch.cuda.stream(st.h2d):
                if self.slot[1] is not None:
                    st.h2d.wait_event(self.slot[1])  # the slot's previous download is done
                prev = st.host_ev.get(self.src.data_ptr())
                if prev is not None:
                    st.h2d.wait_event(prev)  # a pending download into this host bucket lands first
                self.dev.copy_(self.src, non_blocking=True)
            torch.cuda.current_stream(ep.device).wait_stream(st.h2d)
            self.view = None
        else:
            if x.dtype != torch.float32:
                raise Error("bucket must be float32")
            self.view = x
            flat = x.reshape(-1) if x.is_contiguous() else None
            if flat is None or flat.data_ptr() % 16:
                self.dev = x.reshape(-1).clone()
            else:
                self.dev = flat
            self.n = self.dev.numel()

    def finish(self, blocking: bool) -> None:
        """After the launch on the endpoint's stream."""
        if not self.host:
            if self.dev is not self.view and self.dev.data_ptr() != self.view.data_ptr():
                self.view.copy_(self.dev.view_as(self.view))
            return
        ep = self.ep
        st = ep._staging()
        if blocking or not self.pinned:
            ep.sync()  # raises on a latched error: nothing is written back
            self.src.copy_(self.dev)  # device -> pinned, synchronous
            if not self.pinned:
                if isinstance(self.host_t, torch.Tensor):
                    self.host_t.copy_(self.src.view_as(self.host_t))
                else:
                    np.copyto(self.host_t, self.src.numpy().reshape(np.shape(self.host_t)))
            return
        compute = torch.cuda.current_stream(ep.device)  # the collective was launched here
        with torch.cuda.stream(st.d2h):
            st.d2h.wait_stream(compute)
            self.src.copy_(self.dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st.d2h)
            self.slot[1] = ev
            st.host_ev[self.src.data_ptr()] = ev
        st.pending = True


def _on_device(ep: B200Endpoint):
    """torch.cuda.device(ep.device), skipped when it is already current."""
    return contextlib.nullcontext() if torch.cuda.current_device() == ep.device else torch.cuda.device(ep.device)


def _finish(ep: B200Endpoint, b: _Bucket, blocking: bool) -> None:
    if blocking and not b.host:
        ep.sync()
    b.finish(blocking)


def c_fp_s(ep: B200Endpoint, now: float, x, bucket: int = 0, blocking: bool = True) -> float:
    """Allreduce-equivalent; every rank ends with sum_j x_j folded in fp64 in
    ascending rank order (collectives.hpp:50-52)."""
    b = _Bucket(ep, x)
    with _on_device(ep):
        check(lib.b2_c_fp_s(ep.handle, b.dev.data_ptr(), b.n, bucket, ep.stream()))
        _finish(ep, b, blocking)
    g, me = ep.world_size(), ep.rank()
    if g > 1:
        ep._account(4 * (b.n - owned_partition_len(b.n, g, me)) + (g - 1) * 4 * owned_partition_len(b.n, g, me),
                    2 * (g - 1))
    return now


def c_lp_s(ep: B200Endpoint, now: float, x, codec: Codec, es: ErrorState | None, rng=None,
           bucket: int = 0, blocking: bool = True) -> float:
    """Compressed ScatterReduce with two compression phases
    (collectives.hpp:54-61).  es != None applies error compensation.
    Codec{onebit} is the 1-bit Adam aggregation (algorithms.cpp:141-148)."""
    codec._check_supported(rng)
    b = _Bucket(ep, x)
    g, me = ep.world_size(), ep.rank()
    own = owned_partition_len(b.n, g, me)
    dptr = eptr = 0
    dlen = elen = 0
    if es is not None:
        if es.delta.numel() != b.n:
            raise Error("c_lp_s: delta length does not match bucket length")
        if es.epsilon.numel() != own:
            raise Error("c_lp_s: epsilon length does not match owned partition")
        if es.delta.data_ptr() % 16:
            raise Error("c_lp_s: delta must be 16-byte aligned")
        dptr, dlen = es.delta.data_ptr(), es.delta.numel()
        eptr, elen = (es.epsilon.data_ptr() if own else es.delta.data_ptr()), own
    with _on_device(ep):
        if codec.stochastic():  # one 64-bit seed per call from the caller's generator (codec.cpp:71-74)
            check(lib.b2_c_lp_s_stochastic(ep.handle, b.dev.data_ptr(), b.n, dptr, dlen, eptr, elen,
                                           codec._seed(rng), bucket, ep.stream()))
        else:
            check(lib.b2_c_lp_s(ep.handle, b.dev.data_ptr(), b.n, int(codec.kind), dptr, dlen, eptr, elen, bucket,
                                ep.stream()))
        _finish(ep, b, blocking)
    if g > 1:
        key = ("c_lp_s", int(codec.kind), b.n)
        sent = ep._acct.get(key)
        if sent is None:
            per = lambda m: codec.payload_size(m)  # noqa: E731
            sent = sum(per(partition_range(b.n, g, k)[1]) for k in range(g) if k != me) + (g - 1) * per(own)
            ep._acct[key] = sent
        ep._account(sent, 2 * (g - 1))
    return now


def _node_groups(nodes):
    """Members per node (ascending) and the leaders (lowest member of each
    node, ascending), as hierarchical_c forms them (collectives.cpp:299-310)."""
    by_node: dict = {}
    for r, nd in enumerate(nodes):
        by_node.setdefault(nd, []).append(r)
    members = [by_node[nd] for nd in sorted(by_node)]
    leaders = sorted(m[0] for m in members)
    return members, leaders


def _hier_endpoints(ep: B200Endpoint, nodes):
    """Sub-communicators of one node layout, created once (collectively:
    every rank creates every group in the same order); -> (intra endpoint,
    leader endpoint or None, intra gloo group, my leader's global rank)."""
    cache = ep.__dict__.setdefault("_hier", {})
    key = tuple(nodes)
    if key not in cache:
        import torch.distributed as dist
        members, leaders = _node_groups(nodes)
        me = ep.rank()
        intra = lead = igroup = leader = None
        for m in members:
            grp = dist.new_group(m, backend="gloo")
            if me in m:
                intra = B200Endpoint(m.index(me), len(m), ep.device, bootstrap=TorchBootstrap(grp))
                igroup, leader = grp, m[0]
        grp = dist.new_group(leaders, backend="gloo")
        if me in leaders:
            lead = B200Endpoint(leaders.index(me), len(leaders), ep.device, bootstrap=TorchBootstrap(grp))
        cache[key] = (intra, lead, igroup, leader)
    return cache[key]


def hierarchical_c(ep: B200Endpoint, now: float, x, codec: Codec, es: ErrorState | None = None, rng=None,
                   bucket: int = 0, nodes=None) -> float:
    """Two-level centralized aggregation (collectives.cpp:290-385): members'
    x summed in fp64 at the node leader, leaders aggregate across nodes --
    fp64 partials when the codec is lossless, scatter_reduce_lp (C_LP_S over
    the leader group, with es) otherwise -- and every member ends with its
    leader's result.  nodes[r] = node of rank r (default: ep.node_of, i.e.
    one node).  Blocking.

    One node: the reference sums the members in fp64 in ascending rank order
    from +0.0 and rounds once (collectives.cpp:377-380) -- exactly c_fp_s
    over all ranks (ranks >= 2; one rank: (float)(0.0 + (double)x), i.e.
    D_FP_S over the singleton neighbourhood).

    Several nodes, lossless codec: the reference keeps fp64 partials on the
    wire and adds them leader-partial first, then the other leaders in
    ascending order (collectives.cpp:344-372); here c_fp_s folds all ranks
    in ascending order from +0.0.  The two fp64 sums are equal whenever
    they are exact and otherwise differ by a few fp64 ulps, so the fp32
    results agree to within ONE fp32 ulp (tests/mp_parity.py checks gaussian
    inputs against the reference's order with that tolerance).

    Several nodes, lossy codec: c_fp_s inside the node (every member holds
    its leader's (float) node sum, the reference's order), c_lp_s among the
    leaders (scatter_reduce_lp over the leader group, with es), then the
    leader's values are BROADCAST to the members as plain bytes (the
    reference sends float_bytes(x), collectives.cpp:382-384) -- bit-exact,
    -0.0 included.  The byte broadcast runs over the intra-node
    torch.distributed group (this path's inter-node leg has no transport of
    its own)."""
    codec._check_supported(rng)
    g, me = ep.world_size(), ep.rank()
    nodes = list(nodes) if nodes is not None else [ep.node_of(r) for r in range(g)]
    if len(nodes) != g:
        raise Error("hierarchical: node list does not match the world size")
    members, leaders = _node_groups(nodes)
    if len(leaders) == 1 or codec.lossless():
        if g == 1:
            return d_fp_s(ep, now, x, Topology(TopologyKind.full, 1), 0, ReduceMode.sum, bucket)
        return c_fp_s(ep, now, x, bucket)
    intra, lead, igroup, leader = _hier_endpoints(ep, nodes)
    if intra.world_size() == 1:  # the leader alone: (float)(0.0 + (double)x), -0.0 -> +0.0 as in the reference
        d_fp_s(intra, now, x, Topology(TopologyKind.full, 1), 0, ReduceMode.sum, bucket)
    else:
        c_fp_s(intra, now, x, bucket)
    if lead is not None:
        c_lp_s(lead, now, x, codec, es, rng, bucket)
    # down: the leader's values to its members, as bytes
    import torch.distributed as dist
    b = _Bucket(ep, x)
    if intra.world_size() > 1:
        buf = b.dev.cpu()
        dist.broadcast(buf, src=leader, group=igroup)
        b.dev.copy_(buf.to(b.dev.device))
    _finish(ep, b, True)
    return now


def _neighbors(ep: B200Endpoint, topo: Topology, round_: int):
    if topo.n != ep.world_size():
        raise Error("topology size mismatch")  # collectives.cpp:232
    return topo._neighbors_c(ep.rank(), round_)


def d_fp_s(ep: B200Endpoint, now: float, x, topo: Topology, round_: int, mode: ReduceMode,
           bucket: int = 0, blocking: bool = True) -> float:
    """Neighbourhood sum / average (collectives.hpp:63-66)."""
    arr, m = _neighbors(ep, topo, round_)
    b = _Bucket(ep, x)
    with _on_device(ep):
        check(lib.b2_d_fp_s(ep.handle, b.dev.data_ptr(), b.n, arr, m, int(mode), bucket, ep.stream()))
        _finish(ep, b, blocking)
    ep._account((m - 1) * 4 * b.n, m - 1)
    return now


def d_lp_s(ep: B200Endpoint, now: float, x, topo: Topology, round_: int, codec: Codec, mode: ReduceMode,
           rng=None, bucket: int = 0, blocking: bool = True) -> float:
    """As d_fp_s, every contribution (self included) through Q
    (collectives.hpp:68-72).  Any codec, onebit included."""
    codec._check_supported(rng)
    arr, m = _neighbors(ep, topo, round_)
    b = _Bucket(ep, x)
    with _on_device(ep):
        if codec.stochastic():
            check(lib.b2_d_lp_s_stochastic(ep.handle, b.dev.data_ptr(), b.n, arr, m, int(mode), codec._seed(rng),
                                           bucket, ep.stream()))
        else:
            check(lib.b2_d_lp_s(ep.handle, b.dev.data_ptr(), b.n, arr, m, int(codec.kind), int(mode), bucket,
                                ep.stream()))
        _finish(ep, b, blocking)
    ep._account((m - 1) * codec.payload_size(b.n), m - 1)
    return now
