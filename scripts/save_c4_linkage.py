"""Build C4 on the GPU and save its merge list (for host-stage benchmarking on CPU)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config('C4')
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
idx, ws = ragb.build_index(t)
a, b, h, s = idx.linkage()
np.savez_compressed('gpurun_out/c4_linkage.npz', a=a, b=b, h=h, s=s)
print('saved', idx.stats())
