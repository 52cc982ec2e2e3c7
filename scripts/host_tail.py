"""Host stage (a6-a7) timing on a saved merge list: rb_index_from_linkage over
the C4 contexts and the device's merges (gpurun_out/c4_merges.npz, written by
scripts/save_merges.py on the GPU box).  Build the trace variant first:
    python -m paper_2511_03475_b200.build --variant htrace -DRAGB_HOST_TRACE
    RAGB_LIB=htrace python scripts/host_tail.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2511_03475_b200 import ragb
from synth.workload import config

z = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4_merges.npz")
w = config("C4")
for rep in range(int(os.environ.get("REPS", "3"))):
    t = time.perf_counter()
    idx = ragb.index_from_linkage(w.ids, z["a"], z["b"], z["h"], z["size"])
    print(f"host build {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
    del idx
