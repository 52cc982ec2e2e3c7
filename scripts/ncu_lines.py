"""Per-source-line summary of an ncu report (stall samples, instructions).

    python scripts/ncu_lines.py gpurun_out/x.ncu-rep [top]
"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []
fname = "?"
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue  # SASS rows have an address; line rows have '-'
    def f(name):
        try:
            return float(r[hdr.index(name)])
        except Exception:
            return 0.0
    res.append((f("Warp Stall Sampling (All Samples)"), f("Instructions Executed"), f("Thread Instructions Executed"),
                fname, r[0], r[1]))
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
tt = sum(x[2] for x in res) or 1
print(f"total warp inst {ti:.3e}, thread inst {tt:.3e}")
for s, i, t, fn, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{fn[:18]:>18}:{ln:<4} stall {100*s/ts:5.1f}%  inst {100*i/ti:5.1f}%  thr {100*t/tt:5.1f}%  {src.strip()[:80]}")
