"""memcheck target: one build wide enough (N = 60,000) that the first compaction
runs the single-buffer gather kernel (a 120 KB row of codes)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate
t = torch.from_numpy(generate(60000, 8, 600000, 11).ids.view(np.int32)).cuda()
idx, ws = ragb.build_index(t)
torch.cuda.synchronize()
print("big build ok", idx.stats()["linkage_rounds"], flush=True)
