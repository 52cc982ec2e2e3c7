import os, sys, re
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config("C4")
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
ws = None
for r in range(8):
    idx, ws = ragb.build_index(t, workspace=ws)
    torch.cuda.synchronize()
    s = idx.stats()
    print(r, {k: round(s[k], 2) for k in ("distance_ms", "linkage_ms", "host_ms", "total_ms", "merge_ms")}, flush=True)
    del idx
