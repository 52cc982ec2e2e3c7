"""Small builds for compute-sanitizer (memcheck / racecheck / synccheck): C2 in
code mode with in-place and compacting rounds, a tie-heavy input, variable
lengths (fp32 mode), a long-list K, the intersection linkage, and the
row-sharded build in single-process mode."""
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
for mode in ("1", "0"):
    os.environ["RAGB_INPLACE"] = mode
    run(w.ids[:1500])
os.environ.pop("RAGB_INPLACE")
run(generate(1200, 4, 150, 78).ids)                      # tie-heavy: level cliques (warp path)
run(generate(10000, 3, 100000, 5).ids)                    # mostly disjoint: a level of > 4096 vertices (block path)
v = generate(900, 12, 3000, 31, len_min=2); run(v.ids, v.lens)  # variable lengths (fp32 rounds)
run(generate(700, 50, 2000, 9).ids)                       # long lists
run(generate(600, 10, 2000, 8).ids, linkage=ragb.RB_LINK_INTERSECTION)
t = torch.from_numpy(w.ids[:1200].view(np.int32)).cuda()
db = ragb.DistBuilder(3, 1200, w.K, local=True)
db.build(t); torch.cuda.synchronize()
print("sanitize inputs ok", flush=True)
