"""FlatTensor / BucketArena over device memory (mirror of tensor.hpp:16-86).

flatten() concatenates the member tensors into ONE device arena in
registration order with no gaps (one libb2comm launch per 64 members) and
repoints every member at its slice, so writes through the arena (e.g. a
collective updating the bucket in place) are visible through the members and
vice versa -- "unflatten" is implicit, as in tensor.cpp:63-64.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import Error, check, lib


def _shape_product(shape) -> int:  # tensor.cpp:9-17
    p = 1
    for d in shape:
        if d == 0:
            raise Error("tensor shape has a zero dimension")
        p *= d
    return 0 if len(shape) == 0 else p


class FlatTensor:
    """Contiguous float32 device buffer with shape metadata (tensor.hpp:19-48)."""

    def __init__(self, name: str = "", shape=(), values=None, device=None):
        self._name = name
        self._shape = tuple(int(d) for d in shape)
        if name == "" and (shape or values is not None):
            raise Error("tensor name must be non-empty")
        n = _shape_product(self._shape) if self._shape else 0
        dev = device or torch.device("cuda", torch.cuda.current_device())
        if values is None:
            self._data = torch.zeros(n, dtype=torch.float32, device=dev)
        else:
            v = torch.as_tensor(np.asarray(values, dtype=np.float32) if not isinstance(values, torch.Tensor)
                                else values).to(dev, torch.float32).reshape(-1)
            if v.numel() != n:
                raise Error(f"tensor '{name}': shape/data length mismatch")
            self._data = v.clone()

    def name(self) -> str:
        return self._name

    def shape(self):
        return list(self._shape)

    def size(self) -> int:
        return self._data.numel()

    def data(self) -> torch.Tensor:
        """Flat device view (aliases the arena after flatten)."""
        return self._data

    def span(self) -> torch.Tensor:
        return self._data

    def __getitem__(self, k):
        return self._data[k]

    def __setitem__(self, k, v):
        self._data[k] = v

    def is_view(self) -> bool:
        return self._data._base is not None


@dataclass
class TensorView:
    name: str
    offset: int
    length: int


class BucketArena:
    """One contiguous device allocation backing many tensor views."""

    def __init__(self, storage: torch.Tensor | None = None):
        self._storage = storage if storage is not None else torch.empty(0, dtype=torch.float32)
        self._members: list[TensorView] = []

    def members(self):
        return self._members

    def size(self) -> int:
        return self._storage.numel()

    def data(self) -> torch.Tensor:
        return self._storage

    def span(self) -> torch.Tensor:
        return self._storage

    def as_flat(self, name: str = "arena") -> FlatTensor:
        t = FlatTensor.__new__(FlatTensor)
        t._name = name
        t._shape = (self._storage.numel(),)
        t._data = self._storage[:]
        return t

    @staticmethod
    def flatten(tensors) -> "BucketArena":
        """tensor.cpp:46-68.  Errors on empty lists, zero-length members and
        duplicate names."""
        tensors = list(tensors)
        if not tensors:
            raise Error("flatten: empty tensor list")
        seen = set()
        total = 0
        for t in tensors:
            if t.size() == 0:
                raise Error(f"flatten: zero-length tensor '{t.name()}'")
            if t.name() in seen:
                raise Error(f"flatten: duplicate tensor name '{t.name()}'")
            seen.add(t.name())
            total += t.size()
        dev = tensors[0].data().device
        arena = torch.empty(total, dtype=torch.float32, device=dev)
        count = len(tensors)
        srcs = (C.c_void_p * count)(*[t.data().data_ptr() for t in tensors])
        lens = (C.c_size_t * count)(*[t.size() for t in tensors])
        check(lib.b2_bucket_flatten(srcs, lens, count, arena.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
        out = BucketArena(arena)
        off = 0
        for t in tensors:
            n = t.size()
            out._members.append(TensorView(t.name(), off, n))
            t._data = arena[off:off + n]  # repoint: writes alias both ways
            off += n
        return out
