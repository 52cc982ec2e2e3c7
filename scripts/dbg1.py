import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate
from oracle import oracle_c as oc
for N, K in [(64,5),(2048,20),(5000,20),(20000,20)]:
    w = generate(N, K, 50*N, 1)
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    idx, ws = ragb.build_index(t, flags=ragb.RB_KEEP_ROWS | ragb.RB_SKIP_LINKAGE)
    torch.cuda.synchronize()
    print(N, K, 'dist ok', idx.stats(), flush=True)
    idx, ws = ragb.build_index(t, flags=ragb.RB_KEEP_ROWS)
    torch.cuda.synchronize()
    print(N, K, 'full ok', idx.stats(), flush=True)
