"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (last N launches)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, vi, mi, ii = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name'), hdr.index('ID')
seq = [(int(r[ii]), r[ki].split('(')[0].replace('spava::<unnamed>::', ''), float(r[vi].replace(',', '')))
       for r in rows[hi + 1:] if r[mi] == 'gpu__time_duration.sum']
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for s in seq[-n:]:
    print(f"{s[0]:5d} {s[1]:40s} {s[2] / 1000:9.1f} us")
