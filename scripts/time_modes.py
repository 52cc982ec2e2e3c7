"""Time the C4 build under env variants (RAGB_INPLACE / RAGB_CODES / ...): stage times, best of 3."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config('C4')
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
variants = [dict(x.split('=') for x in v.split(',')) if v else {} for v in sys.argv[1:]] or [{}]
for var in variants:
    for k in ('RAGB_INPLACE', 'RAGB_CODES', 'RAGB_GATHER'):
        os.environ.pop(k, None)
    os.environ.update(var)
    best = None
    for _ in range(3):
        idx, ws = ragb.build_index(t)
        torch.cuda.synchronize()
        st = idx.stats()
        del idx, ws
        if best is None or st['total_ms'] < best['total_ms']:
            best = st
    print(json.dumps({'variant': var, **{k: round(v, 2) if isinstance(v, float) else v for k, v in best.items()}}), flush=True)
