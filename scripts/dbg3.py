import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate, config
N = int(sys.argv[1])
w = config('C4') if N == 100000 else generate(N, 20, 10*N, 1)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
idx, ws = ragb.build_index(t, flags=8)
torch.cuda.synchronize()
print('built', idx.stats(), flush=True)
R = ws.rows
ni, nv = idx.nn()
ni = torch.from_numpy(ni).cuda(); nv = torch.from_numpy(nv).cuda()
B = 4096
bad_sym = 0; bad_nn = 0; bad_rows = []
for i0 in range(0, N, B):
    i1 = min(N, i0 + B)
    blk = R[i0:i1]
    # symmetry vs column block
    for j0 in range(0, N, B):
        j1 = min(N, j0 + B)
        m = (blk[:, j0:j1] != R[j0:j1, i0:i1].T)
        c = int(m.sum())
        if c:
            bad_sym += c
            rr = torch.nonzero(m)[:3]
            bad_rows.append((i0 + int(rr[0,0]), j0 + int(rr[0,1])))
    x = blk.clone()
    x[torch.arange(i1 - i0), torch.arange(i0, i1)] = float('inf')
    mn, am = x.min(dim=1)
    # first index attaining the min
    eq = (x == mn[:, None])
    first = torch.argmax(eq.to(torch.int8), dim=1)
    bn = (mn != nv[i0:i1]) | (first.int() != ni[i0:i1])
    if int(bn.sum()):
        bad_nn += int(bn.sum())
        rr = torch.nonzero(bn)[:3].flatten().tolist()
        print('nn bad rows', [(i0 + r, float(mn[r]), int(first[r]), float(nv[i0+r]), int(ni[i0+r])) for r in rr], flush=True)
print('bad_sym', bad_sym, bad_rows[:10], 'bad_nn', bad_nn, flush=True)
idx2, ws2 = ragb.build_index(t, flags=8)
torch.cuda.synchronize()
print('repeat equal', torch.equal(ws.rows, ws2.rows), flush=True)
