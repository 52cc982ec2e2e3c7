"""Save one C4 build's merge list (a, b, h, size) to gpurun_out/c4_merges.npz."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config("C4")
idx, ws = ragb.build_index(torch.from_numpy(w.ids.view(np.int32)).cuda())
torch.cuda.synchronize()
a, b, h, s = idx.linkage()
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c4_merges.npz", a=a, b=b, h=h, size=s)
print("saved", len(a))
