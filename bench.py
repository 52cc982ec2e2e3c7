#!/usr/bin/env python
"""Benchmark of the RAGBoost context-index build on B200 (BASELINE.json metric:
context-pair distances/s and index build time at N=100k, K=20).

One step = one full index build over one batch of N synthetic contexts: a1
validation, a2-a4 distance rows + fused row NN, a5 complete linkage, a6-a7
tree / prefix-first ordering / schedule (rb_build_index + rb_order_contexts).
value = N(N-1)/2 context pairs per build x builds / time (all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C4] [--no-cpu-baseline]

Multi-GPU (torchrun, one process per GPU; default --multi sharded): ONE index
of the same N contexts, rows of the N x N matrix sharded over the GPUs, the
member rows of every compaction round read from the owning GPU over peer
memory (§8(e)); scaling "strong".  --multi replicas: every rank builds the
index of its own batch (seed + rank), scaling "weak".  Timing: CUDA events on
the launching stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
from concurrent.futures import ThreadPoolExecutor
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_CONTEXT = {"hardware": "NVIDIA A6000", "N": 100_000, "k": 20, "build_s": 869.98,
                 "pairs_per_s_derived": 5.75e6, "cite": "PAPER:677, Table 2c"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8192, help="contexts in the oracle sample")
    ap.add_argument("--multi", default="sharded", choices=["sharded", "replicas"],
                    help="N>1: one index with rows sharded over the GPUs (strong scaling), or one "
                         "independent build per GPU (weak scaling)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_desc(name, w):
    r = w.recipe
    return (f"{name}: N={r['N']} contexts, K={r['K']} docs, pool V={r['V']}, "
            f"{'multi-turn' if r['turns'] > 1 else 'single-turn'}, zipf s={r['s_zipf']}, g={r['g']}, "
            f"omega={r['omega']}, seed={r['seed']}")


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region.  In-process
    NVML on a thread (a polling nvidia-smi process competed with the host
    stage for CPU and driver locks and slowed the measured build by ~20%);
    nvidia-smi is the fallback when NVML is unavailable."""

    NAMES = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
             "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
             "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
             "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index, period_s=0.05):
        import threading
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop_ev = threading.Event()
        self.p = None
        self.t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bits = {nm: getattr(pynvml, attr) for nm, attr in self.NAMES.items()}
            # first queries outside the timed region: on a fresh box the first
            # NVML calls of a process can stall CUDA launches for tens of ms
            for _ in range(2):
                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)

            def loop():
                while not self.stop_ev.is_set():
                    try:
                        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        self.mx.append(float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.reasons.update(nm for nm, b in bits.items() if r & b)
                    except pynvml.NVMLError:
                        pass
                    self.stop_ev.wait(period_s)

            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception:  # no NVML: nvidia-smi fallback
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            try:
                self.p = subprocess.Popen(
                    ["nvidia-smi", f"--id={index}",
                     "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            except FileNotFoundError:
                self.p = None

    def stop(self):
        if self.t is not None:
            self.stop_ev.set()
            self.t.join()
        elif self.p is not None:
            self.p.terminate()
            self.p.wait()
            self.f.flush()
            self.f.seek(0)
            for line in self.f.read().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(self.NAMES, parts[4:8]):
                    if v.lower() in ("active", "1"):
                        self.reasons.add(nm)
            os.unlink(self.f.name)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx), "samples": len(self.sm),
                "reasons": sorted(self.reasons), "sampler": "nvml" if self.t is not None else "nvidia-smi"}


# ------------------------------------------------------------------ oracle timing
def oracle_build_time(ids):
    """The oracle as it stands on a sample: C distances (OpenMP), C NN-chain
    linkage, Python tree / ordering / schedule."""
    from oracle import oracle_c as oc
    from oracle import ragb_oracle as o
    t0 = time.perf_counter()
    d = oc.pairwise_rows(ids, None, 1, 200)
    t1 = time.perf_counter()
    oc.row_nn(d)
    Z = oc.linkage(d)
    t2 = time.perf_counter()
    ctxs = o.validate(ids)
    t = o.build_tree(ctxs, list(zip(*Z)))
    o.offline_order(ctxs, t)
    o.schedule(t.path)
    t3 = time.perf_counter()
    return t3 - t0, {"distance_s": t1 - t0, "linkage_s": t2 - t1, "tree_order_s": t3 - t2}


def cpu_model():
    """Host CPU model (lscpu "Model name", else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(w, n_s):
    from oracle import oracle_c as oc
    ids = np.ascontiguousarray(w.ids[:n_s])
    secs, parts = oracle_build_time(ids)
    pairs = n_s * (n_s - 1) / 2
    return {"value": pairs / secs, "unit": "context-pairs/s", "cores": oc.num_threads(), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"first {n_s} contexts of the workload, full build (a1-a7) once",
            "seconds": secs, "stages_s": parts}


def run_reference(args, ws, rank):
    from synth.workload import config
    if rank != 0:
        return
    w = config(args.config)
    n_s = min(args.cpu_sample, w.N)
    ids = np.ascontiguousarray(w.ids[:n_s])
    for _ in range(args.warmup):
        oracle_build_time(ids)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_build_time(ids)
    el = time.perf_counter() - t0
    from oracle import oracle_c as oc
    pairs = n_s * (n_s - 1) / 2
    value = pairs * args.steps / el
    N, K = w.ids.shape
    line = {"impl": "reference", "metric": f"context-pair distances/s (index build, N={N}, K={K})",
            "value": value, "unit": "context-pairs/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32+f32", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, w) + f"; oracle sample = first {n_s} contexts"},
            "cpu_baseline": {"value": value, "unit": "context-pairs/s", "cores": oc.num_threads(),
                             "kind": "oracle", "cpu_model": cpu_model(), "sample": f"first {n_s} contexts per step"},
            "e2e": {"value": value, "unit": "context-pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def run_ours(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2511_03475_b200 import ragb
    from synth.workload import CONFIGS, config

    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = ws > 1 and args.multi == "sharded"
    replicas = ws > 1 and not sharded
    w = config(args.config, seed=CONFIGS[args.config]["seed"] + 1000 * rank) if replicas else config(args.config)
    N, K = w.ids.shape
    pairs = N * (N - 1) / 2
    ids_dev = torch.from_numpy(w.ids.view(np.int32)).to(dev)
    stream = torch.cuda.current_stream(dev)
    p = ragb.make_params(flags=0, stream=ctypes_stream(stream))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if sharded:
        # one index, rows of the N x N matrix sharded over the ws GPUs (§8(e))
        db = ragb.DistBuilder(ws, N, K, rank=rank, local=False, device=dev)

        def build(ids):
            return db.build(ids, stream=stream)
    else:
        wsp = ragb.Workspace(N, K, p, device=dev)
        # independent builds on every GPU of the node: the host stage's
        # threads share the cores
        tu = {"host_threads": max(1, (os.cpu_count() or 2) // ws - 1)} if ws > 1 else {}
        if os.environ.get("RAGB_BENCH_HOST_THREADS"):
            tu["host_threads"] = int(os.environ["RAGB_BENCH_HOST_THREADS"])
        if os.environ.get("RAGB_BENCH_TRACE"):  # diagnostics: per-round events + worker laps on stderr
            tu["trace"] = 2

        def build(ids):
            return ragb.build_index(ids, workspace=wsp, stream=stream, tuning=tu)[0]

    # the caller's output arrays, reused across builds (page-faulted once)
    ord_out = (np.empty((N, K), dtype=np.uint32), np.empty(N, dtype=np.uint8), np.empty(N, dtype=np.int64))

    def step():
        idx = build(ids_dev)
        idx.order_contexts(out=ord_out)
        return idx

    for _ in range(args.warmup):
        flush.zero_()   # warm too: the first launch of torch's fill kernel loads its module (ms to s)
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = Clocks(local, period_s=float(os.environ.get("RAGB_CLOCKS_PERIOD", "0.05")))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    dbg = os.environ.get("RAGB_BENCH_DEBUG")
    e0.record(stream)
    for _ in range(args.steps):
        ta = time.perf_counter()
        flush.zero_()   # L2 flush between builds (256 MB > 126 MB L2)
        tb = time.perf_counter()
        idx = step()
        tc = time.perf_counter()
        stats.append(idx.stats())
        if dbg:
            print(f"step: flush {1e3 * (tb - ta):.2f} step {1e3 * (tc - tb):.2f} lib {stats[-1]['total_ms']:.2f}",
                  file=sys.stderr, flush=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        ms = allreduce_max(ms, dev)
        dist.barrier()
    ms_seq = ms

    # ---- pipelined builds (the headline): RB_ASYNC_HOST returns once the
    # device stages are done and the host stage (a6-a7) finishes on a library
    # thread, so build i's tree/orders/schedule overlap build i+1's device
    # stages; every build still runs a1-a7 and its orders are read back
    # (order_contexts of build i right after build i+1's device stages) -------
    pipelined = not sharded and not os.environ.get("RAGB_BENCH_SEQUENTIAL")

    def run_pipelined(n, build_fn, finish_fn):
        # finish_fn (wait for the host stage, read the orders back, release
        # the handle) runs on a helper thread while the next build's device
        # stages run; all of them complete inside the caller's timed region
        futs = []
        with ThreadPoolExecutor(max_workers=1) as ex:
            for _ in range(n):
                flush.zero_()
                futs.append(ex.submit(finish_fn, build_fn()))
            for f in futs:
                f.result()

    if pipelined:
        def build_async():
            return ragb.build_index(ids_dev, workspace=wsp, stream=stream, tuning=tu,
                                    flags=ragb.RB_ASYNC_HOST)[0]

        def finish(idx):
            idx.order_contexts(out=ord_out)

        run_pipelined(args.warmup, build_async, finish)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0.record(stream)
        run_pipelined(args.steps, build_async, finish)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if ws > 1:
            ms = allreduce_max(ms, dev)
            dist.barrier()
    clocks = clk.stop()

    # ---- end-to-end through the public API with host buffers -------------
    ids_pin = torch.from_numpy(w.ids.view(np.int32)).pin_memory()

    def e2e_build():
        if sharded:  # host ids -> this rank's device, then the sharded build
            ids_d = ids_pin.to(dev, non_blocking=True)
            return db.build(ids_d, stream=stream)
        return ragb.build_index_host(ids_pin.numpy().view(np.uint32), workspace=wsp, stream=stream, tuning=tu,
                                     flags=ragb.RB_ASYNC_HOST if pipelined else 0)[0]

    def e2e_finish(idx):  # the step's results to the caller's host memory
        out, plen, sched = idx.order_contexts(out=ord_out)
        nn_i, nn_d = idx.nn()
        za = idx.linkage()

    run_pipelined(1, e2e_build, e2e_finish)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    if pipelined:
        run_pipelined(args.steps, e2e_build, e2e_finish)
    else:
        for _ in range(args.steps):
            e2e_finish(e2e_build())
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / args.steps
    if ws > 1:
        e2e_ms = allreduce_max(e2e_ms, dev)

    # ---- NEXT-1: online ordering of new contexts against the built index ---
    online = None
    if not sharded and args.config == "C4":
        from synth.workload import generate
        q = generate(10_000, K, 1_000_000, 4004).ids
        online = {"workload": "10,000 new contexts (K=20, V=1e6, seed 4004) searched + inserted + ordered "
                              "into the C4 index (rb_order_contexts, ids != NULL)"}
        warm = build(ids_dev)  # first use of the online kernel and its buffers (module load, cudaMalloc)
        warm.set_online(1)
        warm.order_new(q[:256])
        del warm
        for mode, key in ((1, "device_root_scores"), (0, "host_only")):
            best = None
            for _ in range(2):  # best of two (fresh index each time)
                oi = build(ids_dev)
                torch.cuda.synchronize()
                oi.set_online(mode)
                t0 = time.perf_counter()
                oi.order_new(q)
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
                del oi
            online[key] = {"contexts_per_s": 10_000 / best}

    if rank != 0:
        return
    mean = {k: statistics.mean(s[k] for s in stats) for k in stats[0]}
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs, copy)" if hbm else "fallback 6650 GB/s (B200_PROFILING.md)"
    hbm = hbm or 6650.0
    # rooflines: the distance kernel (a2-a4) and the linkage compaction kernel
    # (a5, k_merge_rows: every launch reads the live rows of the old matrix and
    # writes the new one); "roofline" is the one with the larger step share
    rows_here = -(-N // ws) if sharded else N  # rows of the distance matrix this rank writes
    codes = bool(mean.get("value_codes", 0))
    # fp32 rows (+ 16-bit value codes in code mode) written + ids read (algorithmic)
    dist_bytes = (6.0 if codes else 4.0) * rows_here * N + 4.0 * N * K
    dist_gbs = dist_bytes / (mean["distance_ms"] * 1e-3) / 1e9
    traffic = load_traffic(args.config)
    # the method's own output alone: fp32 rows (4 B per entry) + ids read
    rows_bytes = 4.0 * rows_here * N + 4.0 * N * K
    roof_dist = {"kernel": "k_dist_tile (a2-a4, distance rows + fused row NN)", "bound": "hbm",
                 "achieved": dist_gbs, "peak": hbm, "unit": "GB/s", "frac": dist_gbs / hbm,
                 "traffic": traffic.get("k_dist_tile") if traffic and not sharded else None, "peak_source": peak_src,
                 "algorithmic_bytes_per_launch": dist_bytes, "launches_per_step": 1,
                 "algorithmic_bytes_note": ("4 B fp32 row + 2 B value code" if codes else "4 B fp32 row") +
                 " per entry + 4 N K B of ids",
                 "fp32_rows_only": {"algorithmic_bytes_per_launch": rows_bytes,
                                    "achieved": rows_bytes / (mean["distance_ms"] * 1e-3) / 1e9,
                                    "frac": rows_bytes / (mean["distance_ms"] * 1e-3) / 1e9 / hbm},
                 "share_of_step": mean["distance_ms"] / ms}
    mb = mean["merge_bytes"] / max(mean["merge_launches"], 1)
    merge_gbs = mean["merge_bytes"] / (mean["merge_ms"] * 1e-3) / 1e9 if mean["merge_ms"] > 0 else 0.0
    # the single-GPU code-mode rounds compact with the gather kernel (compact
    # 32-bit map: k_merge_gather2); the
    # sharded build and the fp32 rounds with the window kernel
    mkern = "k_merge_gather2" if codes and not sharded else "k_merge_rows"
    roof_merge = {"kernel": f"{mkern} (a5, linkage compaction rounds)", "bound": "hbm",
                  "achieved": merge_gbs, "peak": hbm, "unit": "GB/s", "frac": merge_gbs / hbm,
                  "traffic": traffic.get(mkern) if traffic and not sharded else None, "peak_source": peak_src,
                  "algorithmic_bytes_per_launch": mb, "launches_per_step": mean["merge_launches"],
                  "algorithmic_bytes_note": ("2 B (16-bit value code)" if codes else "4 B (fp32)") +
                  " x (live old rows^2 + new rows^2) per launch, averaged",
                  "share_of_step": mean["merge_ms"] / ms}
    if roof_merge["share_of_step"] >= roof_dist["share_of_step"]:
        roofline, roofline_other = roof_merge, roof_dist
    else:
        roofline, roofline_other = roof_dist, roof_merge
    line = {
        "metric": f"context-pair distances/s (index build, N={N}, K={K})",
        "value": pairs * (1 if sharded else ws) / (ms * 1e-3),
        "unit": "context-pairs/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": "u32+f32" + ("+u16codes" if codes else ""), "data": "synthetic",
        "config": {"workload": workload_desc(args.config, w) + ("; rank r uses seed+1000r" if replicas else ""),
                   "l2": "256 MB flush write between builds; per-build working set 80 GB >> 126 MB L2",
                   "parallelism": (f"one index, rows sharded over {ws} GPUs (peer-memory exchange)" if sharded
                                   else f"{ws} independent index builds (one per GPU)")},
        "build_time_ms": ms,
        "execution": ("pipelined: RB_ASYNC_HOST builds, build i's host stage (a6-a7) overlaps build i+1's "
                      "device stages; every build runs a1-a7 and its orders are read back inside the timed region"
                      if pipelined else "sequential builds"),
        "sequential": {"ms_per_step": ms_seq, "value": pairs * (1 if sharded else ws) / (ms_seq * 1e-3),
                       "note": "one build at a time (build + order readback), same K / W"},
        "stages_ms": {k: mean[k] for k in ("validate_ms", "distance_ms", "linkage_ms", "host_ms", "total_ms")},
        "distance_pairs_per_s": pairs / (mean["distance_ms"] * 1e-3),
        "linkage_rounds": mean["linkage_rounds"],
        "roofline": roofline,
        "roofline_other": roofline_other,
        "e2e": {"value": pairs * (1 if sharded else ws) / (e2e_ms * 1e-3), "unit": "context-pairs/s",
                "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(N * K * 4),
                "d2h_bytes_per_step": int(N * 8 + 16 * (N - 1) + 8)},
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
        "clocks": clocks,
        "paper_context": PAPER_CONTEXT,
    }
    if online:
        line["online_order"] = online
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, min(args.cpu_sample, N))
    print(json.dumps(line), flush=True)


def allreduce_max(x, dev):
    """Max over ranks (device tensor with NCCL, host tensor with gloo)."""
    import torch
    import torch.distributed as dist
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ctypes_stream(stream):
    import ctypes
    return ctypes.c_void_p(stream.cuda_stream)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def load_traffic(cfg):
    """dram read+write bytes per launch (per kernel) from the committed
    ncu --set full captures under profiles/, or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(cfg)
    except OSError:
        return None


def main():
    args = parse()
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        if args.impl == "reference":
            if rank != 0:
                return
        else:
            import torch
            # one process per GPU; more ranks than GPUs (a one-GPU check of the
            # multi-process path) share devices and fall back to gloo plumbing
            ngpu = max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local % ngpu)
            dist.init_process_group("nccl" if ws <= ngpu else "gloo")
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    try:
        run_ours(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.destroy_process_group()


if __name__ == "__main__":
    main()
