"""host_ms of repeated C4 builds (host stage inside the real build pipeline)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config('C4')
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
p = ragb.make_params()
ws = ragb.Workspace(w.N, w.K, p)
res = []
for r in range(4):
    idx = ragb.build_index(t, workspace=ws)[0]
    st = idx.stats()
    res.append((round(st['host_ms'], 1), round(st['total_ms'], 1)))
    del idx
print('host_ms,total_ms', res)
