import csv, subprocess, sys
rep=sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows=list(csv.reader(out.splitlines())); res=[]; fname='?'; hdr=None
for r in rows:
    if len(r)>=2 and r[0]=="File Path": fname=r[1].split('/')[-1]; continue
    if r and r[0]=="Line No": hdr=r; continue
    if hdr is None or len(r)<len(hdr) or r[2]!='-': continue
    g=lambda n: float(r[hdr.index(n)] or 0)
    res.append((fname,int(r[0]),g("Instructions Executed"),g("Warp Stall Sampling (All Samples)"),r[1]))
ti=sum(x[2] for x in res); ts=sum(x[3] for x in res)
for f,l,i,s,src in sorted(res, key=lambda x:(x[0],x[1])):
    if i/ti>0.002 or s/ts>0.005: print(f"{f[:14]:>14}:{l:<4} inst {100*i/ti:5.1f}% ({i/4.88e6:7.1f}/wchunk) stall {100*s/ts:5.1f}%  {src.strip()[:70]}")
