#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum csv: per-kernel totals."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
tot = collections.OrderedDict()
cnt = collections.Counter()
seq = []
for r in rows[1:]:
    name = r[ki].split('(')[0].replace('void ', '')
    v = float(r[vi].replace(',', ''))
    seq.append((name, v))
for name, v in seq:
    tot[name] = tot.get(name, 0.0) + v
    cnt[name] += 1
allt = sum(tot.values())
print(f"{len(seq)} launches, total {allt/1e6:.3f} ms")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v/1e6:9.3f} ms {cnt[k]:5d}x  {k}")
if len(sys.argv) > 3:
    pat = sys.argv[3]
    print('sequence of', pat, [round(v / 1e6, 3) for n, v in seq if pat in n])
if len(sys.argv) > 4:
    # the last iteration: kernels after the second-to-last k_tile_finalize / k_apply_deltas
    ends = [i for i, (n, v) in enumerate(seq) if 'finalize' in n or 'apply_deltas' in n]
    if len(ends) >= 2:
        it = seq[ends[-2] + 1:ends[-1] + 1]
        print(f"last iteration: {len(it)} launches, {sum(v for _, v in it)/1e3:.1f} us")
        for n, v in it:
            print(f"  {v/1e3:8.1f} us  {n}")
