"""Multi-process row-sharded build (one process per rank, IPC peer memory,
device barriers).  Run with torchrun; on a one-GPU box every rank uses
cuda:0 (IPC between processes on one device exercises the same path).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/dist_mp_check.py [N]
"""
import os, sys, time, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_03475_b200 import ragb
from synth.workload import generate, config

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
ngpu = torch.cuda.device_count()
torch.cuda.set_device(rank % ngpu)
dist.init_process_group("gloo")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
w = config("C2") if N == 4096 else generate(N, 10, 3 * N, 5)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
db = ragb.DistBuilder(world, w.N, w.K, rank=rank, local=False)
dist.barrier()
t0 = time.time()
idx = db.build(t)
torch.cuda.synchronize()
dt = time.time() - t0
res = (idx.linkage(), idx.order_contexts())
if rank == 0:
    si, ws = ragb.build_index(t)
    ref = (si.linkage(), si.order_contexts())
    ok = all(np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
             for x, y in zip(res[0] + res[1], ref[0] + ref[1]))
    print("world", world, "N", w.N, "identical" if ok else "MISMATCH", "build %.1f ms" % (dt * 1e3), flush=True)
dist.barrier()
dist.destroy_process_group()
