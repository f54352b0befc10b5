"""Gradient bucketing + communication/computation overlap on CUDA streams
(mirror of rcomm's Engine, engine.cpp:36-153).

The reference profiles one unfused iteration on its virtual clock, then packs
layers greedily in BACKWARD order (last layer first) into buckets of at most
`bucket_capacity_bytes` (engine.cpp:76-95; a layer larger than the capacity
gets a bucket of its own; fusion off = one bucket per layer), flattens each
bucket's gradients into one arena (engine.cpp:97-107), and during an iteration
launches a bucket's collective as soon as its *trigger layer* -- the last
member to finish backward -- is done, overlapping the rest of backward.

Here the clock is real: backward runs on the caller's compute stream, each
`layer_done(l)` records an event there, and when l is a bucket's trigger the
bucket's primitive is issued on a dedicated communication stream that first
waits for that event.  Every bucket gets its own bucket id, so the primitives'
windows never alias and several buckets can be in flight.
Gradients live in the per-bucket device arenas (`grad(l)` is a view), so no
copy happens between backward and communication.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from ._lib import Error
from .codec import Codec, CodecKind
from .collectives import B200Endpoint, ReduceMode, Topology, TopologyKind, c_fp_s, c_lp_s, d_fp_s, d_lp_s

DEFAULT_BUCKET_CAPACITY_BYTES = 8 << 20  # engine.hpp:58


@dataclass
class Bucket:
    """engine.hpp Bucket: members in backward order, trigger = last member."""
    id: int
    layers: list = field(default_factory=list)
    trigger_layer: int = 0
    elements: int = 0


def plan_buckets(layer_sizes, capacity_bytes: int = DEFAULT_BUCKET_CAPACITY_BYTES,
                 fusion: bool = True) -> list:
    """Greedy reverse-order packing, engine.cpp:76-95 (fp32: 4 bytes/element)."""
    if len(layer_sizes) == 0:
        raise Error("engine: model has no parameter tensors")  # engine.cpp:40
    cap = capacity_bytes if fusion else 0
    buckets: list = []
    used = 0
    L = len(layer_sizes)
    for i in range(L):
        layer = L - 1 - i
        nbytes = 4 * int(layer_sizes[layer])
        if not buckets or used + nbytes > cap:
            buckets.append(Bucket(id=len(buckets)))
            used = 0
        b = buckets[-1]
        b.layers.append(layer)
        b.trigger_layer = layer
        b.elements += int(layer_sizes[layer])
        used += nbytes
    return buckets


class OverlapEngine:
    """Bucketed gradient communication overlapping backward on CUDA streams.

    primitive: "c_lp_s" (default, MinMaxUInt8), "c_fp_s", "d_fp_s", "d_lp_s".
    Usage per iteration::

        for l in reversed(range(L)):          # backward
            ... write layer l's gradient into eng.grad(l) on the compute stream ...
            eng.layer_done(l)
        eng.finish()                          # compute stream waits for every bucket
    """

    def __init__(self, ep: B200Endpoint, layer_sizes, capacity_bytes: int = DEFAULT_BUCKET_CAPACITY_BYTES,
                 fusion: bool = True, primitive: str = "c_lp_s", codec: Codec | None = None,
                 topology: Topology | None = None, mode: ReduceMode = ReduceMode.average,
                 bucket_base: int = 1 << 20, sm_budget: int | None = None):
        if primitive not in ("c_lp_s", "c_fp_s", "d_fp_s", "d_lp_s"):
            raise Error(f"engine: unknown primitive {primitive}")
        self.ep = ep
        self.primitive = primitive
        self.codec = codec or Codec(CodecKind.uniform8)
        if topology is None and primitive.startswith("d_"):
            topology = Topology(TopologyKind.ring, ep.world_size(), 0)
        self.topology = topology
        self.mode = mode
        self.sizes = [int(s) for s in layer_sizes]
        self.buckets = plan_buckets(self.sizes, capacity_bytes, fusion)
        self.bucket_base = bucket_base
        dev = torch.device("cuda", ep.device)
        # one arena per bucket, members in registration (layer) order
        # (engine.cpp:97-107 flattens the members in bucket order)
        self.arenas = []
        self._view = [None] * len(self.sizes)
        self._bucket_of = [0] * len(self.sizes)
        for b in self.buckets:
            arena = torch.zeros(b.elements, dtype=torch.float32, device=dev)
            off = 0
            for layer in b.layers:
                n = self.sizes[layer]
                self._view[layer] = arena[off:off + n]
                self._bucket_of[layer] = b.id
                off += n
            self.arenas.append(arena)
        # high priority: as backward kernels retire, the scheduler hands their
        # SMs to the communication CTAs first
        self.comm_stream = torch.cuda.Stream(device=dev, priority=-1)
        if sm_budget is not None:  # the SMs communication may take (the rest stay with backward)
            ep.set_sm_budget(sm_budget)
        self.round = 0
        self._pending = 0
        self._done = None

    def grad(self, layer: int) -> torch.Tensor:
        """Layer `layer`'s gradient: a view into its bucket's arena."""
        return self._view[layer]

    def bucket_of(self, layer: int) -> Bucket:
        return self.buckets[self._bucket_of[layer]]

    def layer_done(self, layer: int, stream: torch.cuda.Stream | None = None) -> None:
        """Layer `layer`'s gradient is complete on `stream` (default: current).
        At a trigger layer the bucket's collective is issued on the comm stream
        after an event on `stream` -- it overlaps the rest of backward."""
        b = self.bucket_of(layer)
        if layer != b.trigger_layer:
            return
        ev = torch.cuda.Event()
        ev.record(stream or torch.cuda.current_stream(self.ep.device))
        self.comm_stream.wait_event(ev)
        x = self.arenas[b.id]
        bucket = self.bucket_base + b.id
        with torch.cuda.stream(self.comm_stream):
            if self.primitive == "c_lp_s":
                c_lp_s(self.ep, 0.0, x, self.codec, None, bucket=bucket, blocking=False)
            elif self.primitive == "c_fp_s":
                c_fp_s(self.ep, 0.0, x, bucket=bucket, blocking=False)
            elif self.primitive == "d_fp_s":
                d_fp_s(self.ep, 0.0, x, self.topology, self.round, self.mode, bucket=bucket, blocking=False)
            else:
                d_lp_s(self.ep, 0.0, x, self.topology, self.round, self.codec, self.mode, bucket=bucket,
                       blocking=False)
        self._pending += 1

    def finish(self, stream: torch.cuda.Stream | None = None) -> None:
        """The compute stream waits for every bucket issued this iteration.
        Non-blocking: a device error of this iteration's buckets (non-finite
        gradient, rendezvous timeout) is raised by synchronize(), or by the
        next finish() once this iteration's buckets have completed (the
        reference raises synchronously, codec.cpp:24-27; here the report can
        lag by one iteration)."""
        if self._pending != len(self.buckets):
            raise Error(f"engine: {self._pending} of {len(self.buckets)} buckets issued this iteration")
        if self._done is not None and self._done.query():
            self.ep.poll()  # the previous iteration's buckets are complete: report their errors
        ev = torch.cuda.Event()
        ev.record(self.comm_stream)
        (stream or torch.cuda.current_stream(self.ep.device)).wait_event(ev)
        self._done = ev
        self._pending = 0
        self.round += 1

    def synchronize(self) -> None:
        """Wait for every bucket issued so far and raise a latched device error."""
        if self._done is not None:
            self._done.synchronize()
        self.ep.poll()
