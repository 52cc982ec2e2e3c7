"""First merge where the forced in-place rounds differ from the oracle (small N)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from oracle import oracle_c as oc
from synth.workload import generate
for N, K, V in ((64, 5, 200), (300, 5, 600), (2000, 10, 8000)):
    w = generate(N, K, V, 1)
    Z = oc.linkage(oc.pairwise_rows(w.ids, None, 1, 200))
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    for mode in ('0', '1'):
        os.environ['RAGB_INPLACE'] = mode
        idx, ws = ragb.build_index(t)
        L = idx.linkage()
        bad = [i for i in range(N - 1) if any(L[k][i] != Z[k][i] for k in range(4))]
        print(N, 'mode', mode, 'rounds', idx.stats()['linkage_rounds'], 'mismatches', len(bad), flush=True)
        if bad:
            i = bad[0]
            print('  first', i, 'lib', [L[k][i] for k in range(4)], 'oracle', [Z[k][i] for k in range(4)])
