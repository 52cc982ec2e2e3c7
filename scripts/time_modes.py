"""Time the C4 build under strategy variants (rb_params tuning): stage times,
median of 3.  python scripts/time_modes.py 'inplace=0' 'inplace_weight=64.0' ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_03475_b200 import ragb
from synth.workload import config

w = config("C4")
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
ws = None
for spec in ["default"] + sys.argv[1:]:
    tu = {}
    if spec != "default":
        for kv in spec.split(","):
            k, v = kv.split("=")
            tu[k] = float(v) if "." in v else int(v)
    res = []
    for r in range(6):
        idx, ws = ragb.build_index(t, tuning=tu, workspace=ws)
        torch.cuda.synchronize()
        if r:
            res.append(idx.stats())
        del idx
    med = {k: float(np.median([s[k] for s in res])) for k in ("distance_ms", "linkage_ms", "host_ms", "total_ms")}
    print(spec, {k: round(v, 2) for k, v in med.items()}, "rounds", res[0]["linkage_rounds"], flush=True)
