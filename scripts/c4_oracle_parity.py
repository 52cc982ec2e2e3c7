"""C4 (N = 100,000, K = 20) end to end against the oracle (VERDICT r1 task 1c,
SURVEY §8(d) "linkage parity at C4 falls back to oracle-cpp's linkage over the
GPU-produced rows, after those rows have been verified").

1. GPU build with RB_KEEP_ROWS (rows kept) and in the bench configuration
   (flags = 0, rows consumed): identical merge order and document order.
2. EVERY one of the 1e10 distances of the kept rows is compared bit for bit
   with the C oracle (ro_pairwise_rows, blocks of rows, all host cores), and
   every row NN with ro_row_nn.  So the rows the oracle linkage runs on below
   are the oracle's own rows.
3. The C oracle's NN-chain complete linkage (ro_linkage_nnchain) on those rows
   (in place, 40 GB) == the device merge list (a, b, h bits, size).
4. The Python oracle's build_tree / offline_order / schedule on the oracle's
   merge list == the device paths, ordered contexts, prefix lengths, schedule.

Writes gpurun_out/c4_oracle_parity.json (copied to profiles/ by hand).
Takes ~15 min on a 16-core host; needs ~45 GB of host memory.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import oracle_c as oc
from oracle import ragb_oracle as o
from paper_2511_03475_b200 import ragb as F
from synth.workload import config

T0 = time.time()
log = {"config": "C4: N=100000, K=20, V=1e6, seed=4", "host_threads": oc.num_threads()}


def lap(k):
    log[k + "_s"] = round(time.time() - T0, 1)
    print(f"[{log[k + '_s']:8.1f}s] {k}", flush=True)


w = config("C4")
N, K = w.ids.shape
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
# bench configuration first (rows consumed), then the kept-rows build
idx_b, ws = F.build_index(t, flags=0)
torch.cuda.synchronize()
link_b, ord_b = idx_b.linkage(), idx_b.order_contexts()
log["bench_config_stats"] = idx_b.stats()
del ws
torch.cuda.empty_cache()
idx, ws = F.build_index(t, flags=F.RB_KEEP_ROWS)
torch.cuda.synchronize()
a, b, h, s = idx.linkage()
out, pl, sc = idx.order_contexts()
paths = idx.paths()
nn_i, nn_v = idx.nn()
log["keep_rows_stats"] = idx.stats()
same = all(np.array_equal(x, y) for x, y in zip(link_b + ord_b, (a, b, h, s, out, pl, sc)))
log["bench_config_equals_keep_rows"] = bool(same)
lap("gpu_builds")
rows = np.empty((N, N), dtype=np.float32)
B = 4096
for r0 in range(0, N, B):
    n = min(B, N - r0)
    rows[r0:r0 + n] = ws.rows[r0:r0 + n].cpu().numpy()
del ws
torch.cuda.empty_cache()
lap("rows_d2h")
bad_rows = 0
bad_nn = 0
for r0 in range(0, N, B):
    n = min(B, N - r0)
    ref = oc.pairwise_rows(w.ids, None, 1, 200, row0=r0, nrows=n)
    eq = (ref.view(np.uint32) == rows[r0:r0 + n].view(np.uint32)).all(axis=1)
    bad_rows += int((~eq).sum())
    ri, rv = oc.row_nn(ref, row0=r0)
    bad_nn += int(((ri != nn_i[r0:r0 + n]) | (rv.view(np.uint32) != nn_v[r0:r0 + n].view(np.uint32))).sum())
log["rows_checked"] = N
log["rows_mismatch"] = bad_rows
log["nn_mismatch"] = bad_nn
lap("rows_vs_oracle")
Z = oc.linkage(rows, overwrite=True)
del rows
lap("oracle_linkage")
log["merge_order_equal"] = bool(np.array_equal(a, Z[0]) and np.array_equal(b, Z[1])
                                and np.array_equal(h.view(np.uint32), Z[2].view(np.uint32))
                                and np.array_equal(s, Z[3]))
if not log["merge_order_equal"]:
    diff = np.flatnonzero((a != Z[0]) | (b != Z[1]) | (h.view(np.uint32) != Z[2].view(np.uint32)) | (s != Z[3]))
    log["first_merge_diff"] = int(diff[0])
ctxs = o.validate(w.ids, None)
tr = o.build_tree(ctxs, list(zip(*[z.tolist() for z in Z])))
ordered, plen = o.offline_order(ctxs, tr)
sched = o.schedule(tr.path)
lap("oracle_tree")
log["paths_equal"] = paths == tr.path
log["order_equal"] = all(out[i].tolist() == ordered[i] for i in range(N))
log["prefix_len_equal"] = pl.tolist() == plen
log["schedule_equal"] = sc.tolist() == sched
log["all_equal"] = bool(same and bad_rows == 0 and bad_nn == 0 and log["merge_order_equal"] and log["paths_equal"]
                        and log["order_equal"] and log["prefix_len_equal"] and log["schedule_equal"])
lap("done")
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/c4_oracle_parity.json", "w") as f:
    json.dump(log, f, indent=1, default=float)
print(json.dumps(log, default=float))
sys.exit(0 if log["all_equal"] else 1)
