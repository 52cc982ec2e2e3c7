import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
from oracle import oracle_c as oc
w = config('C4'); N = w.N
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
res = {}
for flags in [8, 0, 8, 0]:
    idx, ws = ragb.build_index(t, flags=flags)
    torch.cuda.synchronize()
    ni, nv = idx.nn()
    i0 = int(np.lexsort((np.arange(N), nv))[0])
    print('flags', flags, 'i0', i0, ni[i0], nv[i0], 'row0', ni[0], nv[0], 'row52507', ni[52507], nv[52507], flush=True)
    if flags in res:
        print('  same nn as earlier same-flags run:', np.array_equal(res[flags][0], ni), np.array_equal(res[flags][1], nv))
    res.setdefault(flags, (ni, nv))
    del ws, idx
    torch.cuda.empty_cache()
a, b = res[8], res[0]
diff = np.flatnonzero((a[0] != b[0]) | (a[1] != b[1]))
print('n rows differing', len(diff), diff[:20])
for r in diff[:5]:
    ref = oc.pairwise_rows(w.ids, None, 1, 200, row0=int(r), nrows=1)
    ri, rv = oc.row_nn(ref, row0=int(r))
    print(r, 'oracle', ri[0], rv[0], 'skip', a[0][r], a[1][r], 'full', b[0][r], b[1][r])
