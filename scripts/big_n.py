"""A build beyond C4 (N = 120,000: the first compaction runs the window kernel,
rows wider than the gather kernel's shared memory): checks it completes and
that the merge list is a valid complete-linkage hierarchy (sizes, heights)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate
N = int(sys.argv[1]) if len(sys.argv) > 1 else 120000
w = generate(N, 20, 10 * N, 7)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
for i in range(2):
    t0 = time.perf_counter(); idx, ws = ragb.build_index(t); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = idx.stats()
    print('N', N, 'build %.1f ms' % ((t1 - t0) * 1e3), {k: round(st[k], 2) for k in ('distance_ms', 'linkage_ms', 'host_ms', 'total_ms')}, 'rounds', st['linkage_rounds'], 'codes', st['value_codes'], flush=True)
    a, b, h, s = idx.linkage()
    assert len(a) == N - 1 and np.all(a < b) and s[-1] == N and np.all(np.diff(h) >= 0), 'invalid merge list'
    del idx, ws
    torch.cuda.empty_cache()
print('ok')
