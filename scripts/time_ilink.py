"""Build time with the intersection-representative linkage (NEXT-3)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config, generate
for name, w in (('C2', config('C2')), ('C5_K20', generate(16384, 20, 200000, 5))):
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        idx, ws = ragb.build_index(t, linkage=ragb.RB_LINK_INTERSECTION)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = idx.stats()
    print(name, 'N', w.N, 'build %.1f ms' % (dt * 1e3), 'linkage_ms %.1f' % st['linkage_ms'],
          'per merge %.2f us' % (st['linkage_ms'] * 1e3 / (w.N - 1)), flush=True)
