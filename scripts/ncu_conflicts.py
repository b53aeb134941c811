#!/usr/bin/env python
"""Top shared-memory bank-conflict instructions from an ncu SASS source csv."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: h.index(k) for k in ('Source', 'Instructions Executed', 'L1 Wavefronts Shared Excessive',
                              'L1 Wavefronts Shared', 'Address', 'Warp Stall Sampling (All Samples)')}
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ix['L1 Wavefronts Shared Excessive']] or 0), int(r[ix['L1 Wavefronts Shared']] or 0),
                     int(r[ix['Instructions Executed']] or 0), int(r[ix['Warp Stall Sampling (All Samples)']] or 0),
                     r[ix['Address']], r[ix['Source']].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print('excess wavefronts total', tot, 'shared wavefronts total', sum(d[1] for d in data))
for d in sorted(data, key=lambda d: -d[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{d[0]:>11d} {d[1]:>11d} exec {d[2]:>10d} smp {d[3]:>6d} {d[4]} {d[5]}")
