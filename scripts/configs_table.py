"""Every BASELINE.json config on one GPU: build stage times (best of 3 after a
warm-up build) and pairs/s -> gpurun_out/configs.json (profiles/r01_configs.json)."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_03475_b200 import ragb  # noqa: E402
from synth.workload import config  # noqa: E402

out = []
cases = [("C1", {}), ("C2", {}), ("C3", {}), ("C4", {})] + [("C5", {"K": k}) for k in (5, 20, 50, 100)]
for name, over in cases:
    w = config(name, **over)
    N, K = w.ids.shape
    t = torch.from_numpy(w.ids.view(np.int32)).cuda()
    tl = None if w.lens is None else torch.from_numpy(w.lens.astype(np.uint8)).cuda()
    best = None
    for i in range(4):
        idx, ws = ragb.build_index(t, tl)
        torch.cuda.synchronize()
        st = idx.stats()
        del idx, ws
        if i and (best is None or st["total_ms"] < best["total_ms"]):
            best = st
    torch.cuda.empty_cache()
    rec = {"config": name, "N": N, "K": K, "variable_lengths": tl is not None,
           **{k: round(v, 3) if isinstance(v, float) else v for k, v in best.items() if k != "merge_bytes"},
           "pairs_per_s": N * (N - 1) / 2 / (best["total_ms"] * 1e-3)}
    out.append(rec)
    print(json.dumps(rec), flush=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "configs.json"), "w"), indent=1)
