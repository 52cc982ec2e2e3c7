# ncu --set full of the long-list distance kernel (C5, K = 50) and the tile kernel at C5 K = 20
mkdir -p gpurun_out
cat > gpurun_out/_c5.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
for K in (20, 50):
    t = torch.from_numpy(config('C5', K=K).ids.view(np.int32)).cuda()
    idx, ws = ragb.build_index(t, flags=ragb.RB_SKIP_LINKAGE); torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none -k regex:"k_dist_tile|k_dist_wide" -o gpurun_out/prof_c5 -f python gpurun_out/_c5.py > gpurun_out/prof_c5.log 2>&1
tail -1 gpurun_out/prof_c5.log
