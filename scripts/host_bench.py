"""Time the host stage (a6-a7) alone from a saved C4 merge list."""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config('C4')
z = np.load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/c4_linkage.npz')
best = 1e9
for r in range(5):
    t = time.perf_counter()
    idx = ragb.index_from_linkage(w.ids, z['a'], z['b'], z['h'], z['s'])
    best = min(best, time.perf_counter() - t)
print('host build best %.1f ms' % (best * 1e3))
