"""Debug: code-mode vs fp32-mode linkage on one input (env RAGB_CODES / RAGB_INPLACE set by caller)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate
N = int(sys.argv[1]); K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = generate(N, K, max(40, 3 * N), 100 + N)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
res = {}
for codes in ("0", "1"):
    os.environ["RAGB_CODES"] = codes
    try:
        idx, ws = ragb.build_index(t)
        res[codes] = idx.linkage()
        print(codes, "ok", idx.stats()["linkage_rounds"], flush=True)
    except Exception as e:
        print(codes, "ERR", e, flush=True)
if len(res) == 2:
    for x, y in zip(res["0"], res["1"]):
        print("equal", np.array_equal(x, y), flush=True)
