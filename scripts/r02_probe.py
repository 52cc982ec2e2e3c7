"""Round-2 probe: box resources, and which inputs reach the block-path level
cliques (> 4096 vertices) and the 1024-thread gather (M > 16K)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
print(subprocess.run("nproc; free -g; lscpu | grep -i 'model name'", shell=True, capture_output=True, text=True).stdout, flush=True)
from paper_2511_03475_b200 import ragb
from synth.workload import generate
os.environ["RAGB_TRACE"] = "1"
for (N, K, V, seed) in [(10000, 3, 100000, 5), (20000, 4, 2000, 41), (20000, 4, 200000, 42), (20000, 3, 100000, 43), (24000, 4, 30000, 44)]:
    w = generate(N, K, V, seed)
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    print(f"=== N={N} K={K} V={V} seed={seed}", flush=True)
    idx, ws = ragb.build_index(t)
    torch.cuda.synchronize()
    del idx, ws
