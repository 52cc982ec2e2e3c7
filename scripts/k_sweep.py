"""C5 K sweep: the distance stage (a2-a4) at N = 16,384 for
K in 5..100 -- device time (CUDA events around the library call, best of 5,
linkage skipped), bytes written, fraction of the measured HBM copy bandwidth,
and the full build time.  Writes gpurun_out/k_sweep.json (copied to profiles/r02_k_sweep.json).

    python scripts/k_sweep.py
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_03475_b200 import ragb  # noqa: E402
from synth.workload import config  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
out = []
for K in (5, 10, 15, 20, 30, 50, 75, 100):
    w = config("C5", K=K)
    N = w.ids.shape[0]
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    best_d, best_b, codes = None, None, 0
    for _ in range(5):
        idx, ws = ragb.build_index(t, flags=ragb.RB_SKIP_LINKAGE)
        st = idx.stats()
        best_d = st["distance_ms"] if best_d is None else min(best_d, st["distance_ms"])
        del idx, ws
    for _ in range(3):
        idx, ws = ragb.build_index(t)
        st = idx.stats()
        best_b = st["total_ms"] if best_b is None else min(best_b, st["total_ms"])
        codes = st["value_codes"]
        del idx, ws
    torch.cuda.empty_cache()
    bytes_skip = 4.0 * N * N + 4.0 * N * K  # fp32 rows (no codes without linkage) + ids
    gbs = bytes_skip / (best_d * 1e-3) / 1e9
    rec = {"K": K, "N": N, "distance_ms": round(best_d, 3), "pairs_per_s": N * (N - 1) / 2 / (best_d * 1e-3),
           "GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 3),
           "kernel": "k_dist_tile" if K <= 32 else ("k_dist_wide" if K <= 128 else "k_dist_rows_nn"), "build_ms": round(best_b, 2),
           "linkage_on_codes": bool(codes)}
    out.append(rec)
    print(json.dumps(rec), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"peak_hbm_gbs": peak, "note": "distance stage with RB_SKIP_LINKAGE (fp32 rows only); build = full "
           "index build (code mode for K <= 32)", "sweep": out},
          open(os.path.join(ROOT, "gpurun_out", "k_sweep.json"), "w"), indent=1)
