"""One build with the per-round linkage trace on stderr (tuning trace=1).
python scripts/trace_build.py [C4|C3|N,K,V,seed] [key=value tuning ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_03475_b200 import ragb
from synth.workload import config, generate

arg = sys.argv[1] if len(sys.argv) > 1 else "C4"
if arg.startswith("C"):
    w = config(arg)
else:
    N, K, V, seed = map(int, arg.split(","))
    w = generate(N, K, V, seed)
tu = {"trace": 1}
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    tu[k] = float(v) if "." in v else int(v)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
idx, ws = ragb.build_index(t)  # warm-up
torch.cuda.synchronize()
del idx
idx, ws = ragb.build_index(t, tuning=tu, workspace=ws)
torch.cuda.synchronize()
print(idx.stats(), flush=True)
