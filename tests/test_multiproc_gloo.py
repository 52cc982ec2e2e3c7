"""N>1 host-side plumbing on CPU with gloo, world_size 2 (the GPU path itself
needs devices): the max-over-ranks timing of bench.py, the exchange of the
row-sharded build's handle blobs, and the shard arithmetic of the library."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2511_03475_b200 import ragb
        # bench.py: every rank reports its own time, the line carries the max
        got = bench.allreduce_max(10.0 + rank, "cpu")
        # handle blobs of every rank reach every rank intact (DistBuilder does this)
        blob = bytes([rank]) * ragb.RB_DIST_HANDLE_BYTES
        blobs = [None] * world
        dist.all_gather_object(blobs, blob)
        ok_blobs = all(b == bytes([r]) * ragb.RB_DIST_HANDLE_BYTES for r, b in enumerate(blobs))
        # shard sizes: every rank asks the library for its buffers
        sizes = []
        for N in (1, 5, 4096, 100_000):
            rb, sb = ragb.ctypes.c_size_t(), ragb.ctypes.c_size_t()
            ragb._check(ragb.lib().rb_dist_workspace_size(world, N, 20, ragb.ctypes.byref(rb), ragb.ctypes.byref(sb)))
            sizes.append((N, rb.value, sb.value))
        q.put((rank, got, ok_blobs, sizes))
    finally:
        dist.destroy_process_group()


def test_world2_plumbing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, ok_blobs, sizes in res:
        assert got == 10.0 + world - 1 and ok_blobs
        for N, rb, sb in sizes:
            S = -(-N // world)  # ceil(N / world) rows per rank
            assert rb == S * N * 4
            assert sb >= 2 * S * ((N + 3) // 4 * 4) * 4  # two shard matrices per rank


def test_dist_needs_a_device():
    """No CPU fallback: the multi-process mode allocates its device barrier."""
    from paper_2511_03475_b200 import ragb
    if ragb.torch_cuda_available():
        pytest.skip("CPU-only check")
    h = ragb.ctypes.c_void_p()
    rc = ragb.lib().rb_dist_create(2, 0, 1, ragb.ctypes.byref(h))
    assert rc == ragb.RB_ECUDA
