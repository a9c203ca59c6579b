"""Average per-kernel duration from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, vi, mi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
acc = defaultdict(list)
for r in rows[hi + 1:]:
    if r[mi] == 'gpu__time_duration.sum':
        acc[r[ki].split('(')[0].replace('spava::<unnamed>::', '')[:60]].append(float(r[vi].replace(',', '')) / 1000)
for k, v in sorted(acc.items(), key=lambda x: -sum(x[1])):
    print(f"{k:60s} n={len(v):4d} avg={sum(v)/len(v):9.1f} us  min={min(v):9.1f}")
