import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate, config
N = int(sys.argv[1]); flags = int(sys.argv[2]); reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = config('C4') if N == 100000 else generate(N, 20, 10*N, 1)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
p = ragb.make_params(flags=flags)
wsp = ragb.Workspace(N, 20, p)
prev = None
for r in range(reps):
    idx, ws = ragb.build_index(t, flags=flags, workspace=wsp)
    torch.cuda.synchronize()
    a, b, h, s = idx.linkage()
    ni, nv = idx.nn()
    i0 = int(np.lexsort((np.arange(N), nv))[0])
    print(r, 'stats', idx.stats(), 'first', a[0], b[0], h[0], 'nnmin', i0, ni[i0], nv[i0], flush=True)
    if prev is not None:
        print('same as prev', all(np.array_equal(x, y) for x, y in zip(prev, (a, b, h, s))), flush=True)
    prev = (a, b, h, s)
