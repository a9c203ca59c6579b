"""Stall-reason totals per SASS opcode from `ncu --page source --csv --print-source sass`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
src = hdr.index('Source')
cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
by = defaultdict(lambda: defaultdict(int))
seen = set()
for r in rows[2:]:
    if len(r) <= max(cols) or r[0] in seen:
        continue
    seen.add(r[0])
    toks = r[src].split()
    op = toks[1] if toks and toks[0].startswith('@') and len(toks) > 1 else (toks[0] if toks else '?')
    op = op.split('.')[0]
    for i in cols:
        try:
            by[op][hdr[i][6:]] += int(r[i] or 0)
        except ValueError:
            pass
tot = sum(sum(v.values()) for v in by.values())
for op, v in sorted(by.items(), key=lambda x: -sum(x[1].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    s = sum(v.values())
    top = sorted(v.items(), key=lambda x: -x[1])[:5]
    print(f"{op:10s} {100*s/tot:5.1f}%  " + "  ".join(f"{k}={100*c/tot:.1f}" for k, c in top))
