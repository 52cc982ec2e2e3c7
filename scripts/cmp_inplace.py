"""The merge order must not depend on the round strategy: compare builds with
in-place rounds disabled / automatic / forced (RAGB_INPLACE=0 / unset / 1)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate, config
cases = [('C4', config('C4').ids), ('N30k', generate(30000, 20, 300000, 7).ids),
         ('N20k_K10', generate(20000, 10, 40000, 8).ids)]
for name, ids in cases:
    t = torch.from_numpy(ids.view(np.int32)).cuda()
    res = {}
    for mode in ('0', None, '1'):
        if mode is None:
            os.environ.pop('RAGB_INPLACE', None)
        else:
            os.environ['RAGB_INPLACE'] = mode
        idx, ws = ragb.build_index(t)
        res[mode] = (idx.linkage(), idx.order_contexts(), idx.stats())
        del idx, ws
        torch.cuda.empty_cache()
    ref = res['0']
    for mode in (None, '1'):
        same = all(np.array_equal(x, y) for x, y in zip(ref[0], res[mode][0])) and \
            all(np.array_equal(x, y) for x, y in zip(ref[1], res[mode][1]))
        print(name, 'mode', mode, 'identical' if same else 'MISMATCH',
              'linkage_ms %.1f vs %.1f' % (res[mode][2]['linkage_ms'], ref[2]['linkage_ms']), flush=True)
