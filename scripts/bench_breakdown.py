"""Host-side breakdown of one bench step (device entry) at C4."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_03475_b200 import ragb
from synth.workload import config
w = config('C4')
N, K = w.ids.shape
dev = torch.device('cuda', 0)
ids_dev = torch.from_numpy(w.ids.view(np.int32)).to(dev)
stream = torch.cuda.current_stream(dev)
p = ragb.make_params()
wsp = ragb.Workspace(N, K, p, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
idx = None
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    flush.zero_()
    t1 = time.perf_counter()
    new, _ = ragb.build_index(ids_dev, workspace=wsp, stream=stream)
    t2 = time.perf_counter()
    new.order_contexts()
    t3 = time.perf_counter()
    st = new.stats()
    t4 = time.perf_counter()
    idx = new  # frees the previous index
    t5 = time.perf_counter()
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print('flush %.1f build %.1f (total_ms %.1f) order %.1f stats %.1f free %.1f sync %.1f' % tuple(
        x * 1e3 if i != 1 else x for i, x in enumerate([t1 - t0, (t2 - t1) * 1e3, st['total_ms'], t3 - t2, t4 - t3, t5 - t4, t6 - t5]))
        if False else 'flush %.1f build %.1f (total_ms %.1f) order %.1f stats %.2f free %.1f sync %.1f ms' % (
        (t1 - t0) * 1e3, (t2 - t1) * 1e3, st['total_ms'], (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3,
        (t6 - t5) * 1e3), flush=True)
