#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into a committed JSON/text profile.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_<name> [--kernel REGEX]

Writes <out>.json (per-kernel key metrics) and <out>.txt (human summary).
"""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    kern = None
    if "--kernel" in sys.argv:
        kern = sys.argv[sys.argv.index("--kernel") + 1]
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", "regex:" + kern] if kern else [])
    rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True, check=True).stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    lines = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name"), "metrics": {}}
        for k in KEYS:
            if k in d:
                ent["metrics"][k] = {"value": d[k], "unit": u.get(k, "")}
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): d[k]
                  for k in d if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:6]
        ent["top_stalls_per_issue"] = dict(top)
        res.append(ent)
        lines.append(f"== {ent['kernel']}")
        for k, v in ent["metrics"].items():
            lines.append(f"   {k:60s} {v['value']} {v['unit']}")
        lines.append("   stalls/issue: " + ", ".join(f"{k}={v}" for k, v in top))
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    with open(out + ".txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
