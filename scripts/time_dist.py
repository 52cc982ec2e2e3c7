"""Distance stage alone (a1-a4, RB_SKIP_LINKAGE) at C4 or a C5 K: median of
several builds.  python scripts/time_dist.py [C4|K=<k>] [reps] [codes]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_03475_b200 import ragb
from synth.workload import config

arg = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = config("C4") if arg == "C4" else config("C5", K=int(arg.split("=")[1]))
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
flags = ragb.RB_SKIP_LINKAGE if "skip" in sys.argv else 0  # full build: the distance kernel also writes codes
p = ragb.make_params(flags=flags, stream=ragb._stream_ptr(None))
ws = ragb.Workspace(w.N, w.K, p)
ms = []
for r in range(reps + 1):
    idx, _ = ragb.build_index(t, flags=flags, workspace=ws)
    torch.cuda.synchronize()
    if r:
        ms.append(idx.stats()["distance_ms"])
N = w.N
print(f"{arg} N={N} K={w.K} distance_ms median {np.median(ms):.3f} min {min(ms):.3f}  "
      f"fp32 rows {4*N*N/np.median(ms)/1e6:.0f} GB/s", flush=True)
