"""§8(e) row-sharded build with ONE PROCESS PER RANK on the GPU (the
multi-process mode: CUDA IPC mappings of every rank's buffers, device
barriers on peer counters, torch.distributed (gloo) for the handle blobs).
Two ranks; on a one-GPU box both processes share cuda:0 (IPC between
processes on one device runs the same code path).  Peer access between the
GPUs is checked up front.  Every rank's merge order, NN, document order,
schedule and paths must equal the single-GPU build's bit for bit (which the
other GPU tests pin to the oracle)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(name):
    from synth.workload import config, generate
    if name == "C2":
        w = config("C2")
        return w.ids, None
    if name == "ties":
        return generate(3000, 4, 300, 32).ids, None
    w = generate(2053, 12, 5000, 77, len_min=3)
    return w.ids, w.lens


def _worker(rank, world, port, name, outdir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_2511_03475_b200 import ragb
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids, lens = _case(name)
        t = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
        tl = None if lens is None else torch.from_numpy(lens).cuda()
        db = ragb.DistBuilder(world, ids.shape[0], ids.shape[1], rank=rank, local=False)
        dist.barrier()
        idx = db.build(t, tl)
        torch.cuda.synchronize()
        a, b, h, s = idx.linkage()
        ni, nv = idx.nn()
        out, pl, sc = idx.order_contexts()
        paths = np.array([x for p in idx.paths() for x in ([len(p)] + p)], dtype=np.int64)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), a=a, b=b, h=h, s=s, ni=ni, nv=nv, out=out, pl=pl, sc=sc,
                 paths=paths)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C2", "ties", "var"])
def test_row_sharded_two_processes(name, tmp_path):
    import torch.multiprocessing as mp
    from paper_2511_03475_b200 import ragb
    ngpu = torch.cuda.device_count()
    if ngpu >= 2:
        assert torch.cuda.can_device_access_peer(0, 1), \
            "GPUs 0 and 1 have no peer access: the row-sharded build reads peer memory"
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    ids, lens = _case(name)
    t = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tl = None if lens is None else torch.from_numpy(lens).cuda()
    si, ws = ragb.build_index(t, tl)
    a, b, h, s = si.linkage()
    ni, nv = si.nn()
    out, pl, sc = si.order_contexts()
    paths = np.array([x for p in si.paths() for x in ([len(p)] + p)], dtype=np.int64)
    ref = dict(a=a, b=b, h=h, s=s, ni=ni, nv=nv, out=out, pl=pl, sc=sc, paths=paths)
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        for k, v in ref.items():
            assert np.array_equal(np.asarray(got[k]).view(np.uint8), np.asarray(v).view(np.uint8)), (r, k)
