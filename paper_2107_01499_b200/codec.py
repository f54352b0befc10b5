"""Codec / ErrorState / compensate_encode over device memory.

Mirror of rcomm's codec.hpp:13-54.  The uniform8 ("MinMaxUInt8") encode and
decode run in libb2comm's sm_100a kernels; the wire payload is the exact
reference layout ``[min f32][max f32][u8 x N]`` (codec.hpp:21-24) held in a
device uint8 tensor.  Host inputs (numpy arrays / CPU tensors) are staged to
the GPU and the payload / result is copied back, so the reference's own tests
can drive this class unchanged.
"""
from __future__ import annotations

import ctypes as C
import enum

import numpy as np
import torch

from . import _lib
from ._lib import Error, check, lib


class CodecKind(enum.IntEnum):
    identity = _lib.CODEC_IDENTITY
    uniform8 = _lib.CODEC_UNIFORM8
    onebit = _lib.CODEC_ONEBIT


class Rounding(enum.IntEnum):
    nearest = 0
    stochastic = 1


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _as_device(x, device=None):
    """-> (device tensor, host original or None)."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x, None
    t = torch.as_tensor(np.asarray(x, dtype=np.float32) if not isinstance(x, torch.Tensor) else x)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return t.to(dev, dtype=torch.float32).contiguous(), x


def _aligned(t: torch.Tensor) -> bool:
    return t.data_ptr() % 16 == 0


class Codec:
    """Lossy compression function Q (codec.hpp:25-36).  Immutable."""

    def __init__(self, kind: CodecKind = CodecKind.identity, rounding: Rounding = Rounding.nearest):
        self.kind = CodecKind(kind)
        self.rounding = Rounding(rounding)

    def __repr__(self) -> str:
        return f"Codec({self.kind.name}, {self.rounding.name})"

    def lossless(self) -> bool:
        return self.kind == CodecKind.identity

    def payload_size(self, n: int) -> int:
        """codec.cpp:31-38 (cached per length: the per-call host cost matters for small buckets)."""
        cache = self.__dict__.setdefault("_psize", {})
        v = cache.get(n)
        if v is None:
            v = cache[n] = int(lib.b2_payload_size(int(self.kind), n))
        return v

    def _check_supported(self, rng, collective: bool = True) -> None:
        if self.stochastic() and rng is None:  # codec.cpp:70 wording
            raise Error("uniform8 stochastic rounding needs a generator")

    def stochastic(self) -> bool:
        """uniform8 with Rounding::stochastic (codec.cpp:67-78)."""
        return self.kind == CodecKind.uniform8 and self.rounding == Rounding.stochastic

    @staticmethod
    def _seed(rng) -> int:
        """64 bits drawn from the caller's generator (random.Random-like or a
        numpy Generator), advancing it like the reference's per-element draws
        advance its mt19937 (codec.cpp:71-74)."""
        if hasattr(rng, "getrandbits"):
            return int(rng.getrandbits(64))
        if hasattr(rng, "integers"):
            return int(rng.integers(0, 2**64, dtype=np.uint64))
        raise Error("stochastic rounding: rng must provide getrandbits() or integers()")

    # -- SoA device form (what the collectives use internally) -------------
    def encode_soa(self, x: torch.Tensor, seed: int | None = None):
        """uniform8: -> (codes uint8[n], hdr float32[4]) on x's device; raises
        Error on non-finite input (codec.cpp:24-27).  seed: stochastic rounding."""
        assert x.is_cuda and x.dtype == torch.float32
        x = x.contiguous()
        if not _aligned(x):
            x = x.clone()
        n = x.numel()
        codes = torch.empty(max(n, 4) + 16, dtype=torch.uint8, device=x.device)
        hdr = torch.empty(4, dtype=torch.float32, device=x.device)
        if seed is None:
            check(lib.b2_u8_encode(x.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(), _stream(x.device)))
        else:
            check(lib.b2_u8_encode_stochastic(x.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(), seed,
                                              _stream(x.device)))
        lohi = hdr[:2].cpu()
        if not bool(torch.isfinite(lohi).all()):
            raise Error("encode: non-finite input value")
        return codes[:n], hdr

    def decode_soa(self, codes: torch.Tensor, hdr: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        n = out.numel()
        if n == 0:
            return out
        c = codes if codes.data_ptr() % 16 == 0 else codes.clone()
        o = out if _aligned(out) and out.is_contiguous() else torch.empty_like(out)
        check(lib.b2_u8_decode(c.data_ptr(), hdr.data_ptr(), n, o.data_ptr(), _stream(out.device)))
        if o is not out:
            out.copy_(o)
        return out

    # -- wire form (codec.hpp:32-35) ----------------------------------------
    def encode(self, x, rng=None):
        """Payload bytes.  Device input -> device uint8 tensor; host input ->
        numpy uint8 array (the reference's Payload)."""
        self._check_supported(rng, collective=False)
        xd, host = _as_device(x)
        xd = xd.reshape(-1)
        n = xd.numel()
        if self.kind == CodecKind.onebit:  # codec.cpp:81-88
            if not _aligned(xd):
                xd = xd.clone()
            wire = torch.empty(((4 + (n + 7) // 8) + 15) // 16 * 16, dtype=torch.uint8, device=xd.device)
            check(lib.b2_onebit_encode(xd.data_ptr() if n else 0, n, wire.data_ptr(), _stream(xd.device)))
            wire = wire[:self.payload_size(n)]
            if bool(torch.isnan(wire[:4].view(torch.float32)).all()):  # the kernel's non-finite mark
                raise Error("encode: non-finite input value")  # codec.cpp:24-27
            return wire.cpu().numpy() if host is not None else wire
        if self.kind == CodecKind.identity:
            if n and not bool(torch.isfinite(xd).all()):
                raise Error("encode: non-finite input value")
            wire = xd.contiguous().view(torch.uint8).clone()
        else:
            stochastic = self.rounding == Rounding.stochastic
            codes, hdr = self.encode_soa(xd, self._seed(rng) if stochastic else None)
            wire = torch.empty(8 + n, dtype=torch.uint8, device=xd.device)
            check(lib.b2_u8_pack_wire(codes.data_ptr() if n else 0, hdr.data_ptr(), n, wire.data_ptr(),
                                      _stream(xd.device)))
        return wire.cpu().numpy() if host is not None else wire

    def decode(self, payload, n_or_out):
        """decode(payload, n) -> new buffer; decode(payload, out) -> fills out."""
        host = not (isinstance(payload, torch.Tensor) and payload.is_cuda)
        if isinstance(n_or_out, (int, np.integer)):
            n, out = int(n_or_out), None
        else:
            out = n_or_out
            n = out.numel() if isinstance(out, torch.Tensor) else np.asarray(out).size
        size = payload.numel() if isinstance(payload, torch.Tensor) else len(payload)
        if size != self.payload_size(n):  # codec.cpp:96-97
            raise Error("decode: malformed payload (length mismatch)")
        dev = payload.device if not host else torch.device("cuda", torch.cuda.current_device())
        p = payload if not host else torch.as_tensor(np.asarray(payload, dtype=np.uint8)).to(dev)
        res = torch.empty(n, dtype=torch.float32, device=dev)
        if n and self.kind == CodecKind.onebit:  # codec.cpp:110-114
            w = torch.zeros(((size + 15) // 16) * 16, dtype=torch.uint8, device=dev)
            w[:size].copy_(p.reshape(-1))
            check(lib.b2_onebit_decode(w.data_ptr(), n, res.data_ptr(), _stream(dev)))
        elif n:
            if self.kind == CodecKind.identity:
                res.copy_(p.contiguous().view(torch.float32))
            else:
                codes = torch.empty(n + 16, dtype=torch.uint8, device=dev)
                hdr = torch.empty(4, dtype=torch.float32, device=dev)
                check(lib.b2_u8_unpack_wire(p.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(), _stream(dev)))
                self.decode_soa(codes, hdr, res)
        if out is None:
            return res.cpu().numpy() if host else res
        if isinstance(out, torch.Tensor):
            out.copy_(res.view_as(out))
        else:
            out[...] = res.cpu().numpy().reshape(np.shape(out))
        return out


class ErrorState:
    """Worker-side delta (bucket length) and owner-side epsilon (owned
    partition length), zero-initialised (codec.hpp:38-47); device tensors."""

    def __init__(self, bucket_len: int = 0, owned_len: int = 0, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.delta = torch.zeros(bucket_len, dtype=torch.float32, device=dev)
        self.epsilon = torch.zeros(owned_len, dtype=torch.float32, device=dev)


def compensate_encode(codec: Codec, x, delta, rng=None, decoded: list | None = None):
    """codec.hpp:49-54 / codec.cpp:125-137: encodes Q(x - delta) and replaces
    delta by the exact residual (x - delta) - D(Q(x - delta))."""
    codec._check_supported(rng)
    xd, host = _as_device(x)
    n = xd.numel()
    host_delta = not (isinstance(delta, torch.Tensor) and delta.is_cuda)
    dd = torch.as_tensor(np.asarray(delta, dtype=np.float32)).to(xd.device) if host_delta else delta
    if dd.numel() != n:
        raise Error("compensate_encode: length mismatch")
    if codec.kind == CodecKind.identity:  # y = x - delta is the payload; delta = y - y (one kernel)
        xa = xd.reshape(-1).contiguous()
        da = dd.reshape(-1) if dd.is_contiguous() else dd.reshape(-1).clone()
        dec = torch.empty(n, dtype=torch.float32, device=xd.device)
        flag = torch.zeros(1, dtype=torch.int32, device=xd.device)
        check(lib.b2_identity_compensate_encode(xa.data_ptr() if n else 0, da.data_ptr() if n else 0, n,
                                                dec.data_ptr() if n else 0, flag.data_ptr(), _stream(xd.device)))
        if int(flag.item()):
            raise Error("encode: non-finite input value")  # codec.cpp:24-27, delta untouched
        if da.data_ptr() != dd.data_ptr():
            dd.copy_(da.view_as(dd))
        payload = dec.view(torch.uint8).clone()
    elif codec.kind == CodecKind.onebit:  # y = x - delta; P = Q(y); delta = y - D(P), all exact fp32
        xa = xd.reshape(-1) if _aligned(xd) and xd.is_contiguous() else xd.reshape(-1).clone()
        da = dd.reshape(-1).clone()  # written only once the encode succeeded
        dec = torch.empty(max(n, 4), dtype=torch.float32, device=xd.device)[:n]
        wire = torch.empty(((4 + (n + 7) // 8) + 15) // 16 * 16, dtype=torch.uint8, device=xd.device)
        check(lib.b2_onebit_compensate_encode(xa.data_ptr() if n else 0, da.data_ptr() if n else 0, n,
                                              wire.data_ptr(), dec.data_ptr(), _stream(xd.device)))
        payload = wire[:codec.payload_size(n)]
        if bool(torch.isnan(payload[:4].view(torch.float32)).all()):  # the kernel's non-finite mark
            raise Error("encode: non-finite input value")
        dd.copy_(da.view_as(dd))
    else:
        xa = xd if _aligned(xd) else xd.clone()
        da = dd if _aligned(dd) and dd.is_contiguous() else dd.clone()
        codes = torch.empty(max(n, 4) + 16, dtype=torch.uint8, device=xd.device)
        hdr = torch.empty(4, dtype=torch.float32, device=xd.device)
        dec = torch.empty(n, dtype=torch.float32, device=xd.device)
        check(lib.b2_u8_compensate_encode(xa.data_ptr(), da.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(),
                                          dec.data_ptr() if n else 0, _stream(xd.device)))
        if not bool(torch.isfinite(hdr[:2]).all()):
            raise Error("encode: non-finite input value")
        if da is not dd:
            dd.copy_(da)
        payload = torch.empty(8 + n, dtype=torch.uint8, device=xd.device)
        check(lib.b2_u8_pack_wire(codes.data_ptr(), hdr.data_ptr(), n, payload.data_ptr(), _stream(xd.device)))
    if host_delta:
        np.copyto(np.asarray(delta), dd.cpu().numpy())
    if decoded is not None:
        decoded[:] = [dec.cpu().numpy() if host else dec]
    return payload.cpu().numpy() if host else payload
