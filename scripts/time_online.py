"""NEXT-1 throughput: M new contexts into the C4 index, root scores on the
device (set_online(1)) vs on the host (set_online(0))."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_03475_b200 import ragb
from synth.workload import config, generate

w = config("C4")
M = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
q = generate(M, 20, 1_000_000, 4004).ids
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
for mode in (1, 0, 1):
    idx, ws = ragb.build_index(t, tuning=dict(trace=1 if len(sys.argv) > 2 else 0))
    torch.cuda.synchronize()
    idx.set_online(mode)
    t0 = time.perf_counter()
    idx.order_new(q)
    dt = time.perf_counter() - t0
    print(f"mode {mode}: {M} queries {dt*1e3:.1f} ms  {M/dt:.0f} contexts/s", flush=True)
    del idx, ws
