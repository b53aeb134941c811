#!/usr/bin/env python
"""Group an ncu SASS source page (csv) into straight-line blocks by execution count."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index('Instructions Executed'); src = h.index('Source'); smp = h.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows[2:]:
    try: data.append((int(r[ie]), int(r[smp]), r[0], r[src]))
    except Exception: pass
tot = sum(d[0] for d in data) or 1; tots = sum(d[1] for d in data) or 1
print('total inst', tot, 'samples', tots)
blocks, cur = [], None
for d in data:
    if cur and d[0] == cur[0]:
        cur[1] += 1; cur[2] += d[1]; cur[3].append(d[3])
    else:
        cur = [d[0], 1, d[1], [d[3]]]; blocks.append(cur)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 14
full = len(sys.argv) > 3
for b in sorted(blocks, key=lambda b: -b[0] * b[1])[:n]:
    print(f"exec {b[0]:>10d} x {b[1]:3d} = {b[0]*b[1]/tot*100:5.1f}% inst, {b[2]/tots*100:5.1f}% smp | " +
          ('\n      ' + '\n      '.join(x.strip() for x in b[3]) if full else ' ; '.join(x.strip()[:26] for x in b[3][:6])))
