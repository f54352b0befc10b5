"""Host-side multi-process logic on CPU (world_size 2, 4 and 8, gloo): the
window-handle bootstrap that b2_comm_create's allgather hook runs through
(TorchBootstrap), the in-process ThreadBootstrap, and the callback marshalling
of B200Endpoint._allgather."""
import ctypes as C
import os
import socket
import threading

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2107_01499_b200.collectives import B200Endpoint, TorchBootstrap
        bs = TorchBootstrap()
        blob = bytes([rank]) * 7 + b"\x00" * 81  # 88 bytes, like the window Blob
        parts = bs.allgather(blob, world)
        ok = parts == [bytes([r]) * 7 + b"\x00" * 81 for r in range(world)]
        # the C-callback marshalling, without a device: call _allgather directly
        ep = B200Endpoint.__new__(B200Endpoint)
        ep._rank, ep._world, ep._bootstrap = rank, world, bs
        send = C.create_string_buffer(blob, len(blob))
        recv = C.create_string_buffer(len(blob) * world)
        rc = ep._allgather(None, C.addressof(send), len(blob), C.addressof(recv))
        ok = ok and rc == 0 and recv.raw == b"".join(bytes([r]) * 7 + b"\x00" * 81 for r in range(world))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_torch_bootstrap_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]


def test_thread_bootstrap():
    from paper_2107_01499_b200.collectives import ThreadBootstrap
    world = 4
    bs = ThreadBootstrap(world)
    out = [None] * world

    def run(r):
        out[r] = [bs.allgather(bytes([r, i]), world, r) for i in range(3)]

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for r in range(world):
        for i in range(3):
            assert out[r][i] == [bytes([k, i]) for k in range(world)]
