"""Where does a bench step's time go: build / order_contexts / flush (wall clock, synced)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config('C4'); N, K = w.ids.shape
dev = torch.device('cuda', 0)
ids = torch.from_numpy(w.ids.view(np.int32)).to(dev)
st = torch.cuda.current_stream(dev)
import ctypes
p = ragb.make_params(flags=0, stream=ctypes.c_void_p(st.cuda_stream))
wsp = ragb.Workspace(N, K, p, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    flush.zero_(); torch.cuda.synchronize(); t1 = time.perf_counter()
    idx = ragb.build_index(ids, workspace=wsp, stream=st)[0]; torch.cuda.synchronize(); t2 = time.perf_counter()
    idx.order_contexts(); t3 = time.perf_counter()
    s = idx.stats(); t4 = time.perf_counter()
    del idx; t5 = time.perf_counter()
    print('flush %.1f build %.1f order %.1f stats %.1f free %.1f (lib total %.1f)' % tuple(
        [1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)] + [s['total_ms']]), flush=True)
