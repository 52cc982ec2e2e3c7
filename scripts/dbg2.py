import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import generate, config
N = int(sys.argv[1]); flags = int(sys.argv[2])
w = config('C4') if N == 100000 else generate(N, 20, 10*N, 1)
t = torch.from_numpy(w.ids.view(np.int32)).cuda()
idx, ws = ragb.build_index(t, flags=flags)
torch.cuda.synchronize()
print(N, flags, 'ok', idx.stats(), flush=True)
