"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck) that
reach every kernel family: the distance tile kernel (TMA rings), code-mode
rounds in place and compacting, the warp-resident level cliques, the vertex
sweep with helper CTAs (a level above 4096 vertices), variable lengths (fp32
rounds, general distance kernel), long lists, the intersection linkage, the
row-sharded build in single-process mode and the online root-score kernel."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_03475_b200 import ragb
from synth.workload import config, generate


def run(ids, lens=None, **kw):
    t = torch.from_numpy(np.ascontiguousarray(ids).view(np.int32)).cuda()
    tl = None if lens is None else torch.from_numpy(np.ascontiguousarray(lens, dtype=np.uint8)).cuda()
    idx, ws = ragb.build_index(t, tl, **kw)
    torch.cuda.synchronize()
    return idx


w = config("C2")
for mode in (1, 0):
    run(w.ids[:1500], tuning=dict(inplace=mode))
run(w.ids[:1500], tuning=dict(gather=0))                  # window compaction on codes
run(generate(1200, 4, 150, 78).ids)                       # tie-heavy: level cliques (warp path)
run(generate(10000, 3, 100000, 5).ids)                    # a level of > 4096 vertices (sweep + helper CTAs)
v = generate(900, 12, 3000, 31, len_min=2); run(v.ids, v.lens)  # variable lengths (fp32 rounds)
run(generate(700, 50, 2000, 9).ids)                       # long lists
run(generate(600, 10, 2000, 8).ids, linkage=ragb.RB_LINK_INTERSECTION)
t = torch.from_numpy(w.ids[:1200].view(np.int32)).cuda()
db = ragb.DistBuilder(3, 1200, w.K, local=True)
db.build(t); torch.cuda.synchronize()
idx = run(w.ids)
idx.set_online(1)
idx.order_new(generate(300, 10, 20000, 99).ids)           # online root scores
print("sanitize inputs ok", flush=True)
