"""Summarise an ncu launch list (gpu__time_duration.sum csv): totals per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[h]
ki, vi, ii = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('ID')
seq = [(int(r[ii]), r[ki].split('(')[0].replace('ragb::<unnamed>::', '').replace('void ', ''),
        float(r[vi].replace(',', '')) / 1e3) for r in rows[h + 1:] if len(r) > vi]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for _, k, v in seq:
    tot[k] += v
    cnt[k] += 1
S = sum(tot.values())
for k in sorted(tot, key=lambda k: -tot[k]):
    print("%-44s launches=%4d total=%9.3f ms share=%5.1f%%" % (k[:44], cnt[k], tot[k] / 1e3, 100 * tot[k] / S))
print("sum of kernel time %.3f ms over %d launches" % (S / 1e3, len(seq)))
if len(sys.argv) > 2:
    for i, k, v in seq:
        if sys.argv[2] in k:
            print(i, k, "%.1f us" % v)
