"""Per-kernel DRAM traffic per launch from an ncu --set full report ->
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).

    python scripts/traffic_json.py gpurun_out/prof_full.ncu-rep C4
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[2:]:
        name = next((k for k in ("k_dist_tile", "k_merge_rows", "k_merge_gather2", "k_merge_gather") if k in r[ki]), None)
        if name is None:
            continue
        b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
        per.setdefault(name, []).append(b)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
    except OSError:
        d = {}
    d[cfg] = {k: sum(v) / len(v) for k, v in per.items()}
    d[cfg + "_launches"] = {k: len(v) for k, v in per.items()}
    d["_source"] = ("ncu --set full --clock-control none of scripts/dbg2.py (one C4 build): "
                    "dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over the kernel's launches")
    json.dump(d, open(path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
