#!/usr/bin/env python
"""Print the hottest SASS loop of an ncu source page (csv from
`ncu -i REP --page source --csv --print-source sass`): the longest contiguous
run of instructions whose executed count equals the modal count among the
most-executed instructions, with per-instruction stall-sample shares.
usage: ncu_hot_loop.py SASS_CSV [CANDIDATES_PER_PASS]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
per_pass = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hdr = rows[1]
ia, isrc, ismp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("# Samples"), hdr.index("Instructions Executed")
ins = [(r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)) for r in rows[2:] if len(r) > iex]
tot_s = sum(x[1] for x in ins) or 1
tot_i = sum(x[2] for x in ins) or 1
# modal executed count weighted by instruction count * executed count
w = collections.Counter()
for _, _, e in ins:
    w[e] += e
mode = max(w, key=w.get)
best, cur = (0, 0), None
for k, x in enumerate(ins + [("", 0, -1)]):
    if x[2] == mode:
        cur = k if cur is None else cur
    elif cur is not None:
        if k - cur > best[1] - best[0]:
            best = (cur, k)
        cur = None
a, b = best
n = sum(1 for x in ins if x[2] == mode)
print(f"{rows[0][1]}")
print(f"hot loop body: {n} SASS instructions executed {mode} times each (one pass = {per_pass} candidates per lane: "
      f"{n / per_pass:.1f} instructions per candidate slot); share of all warp instructions "
      f"{100.0 * n * mode / tot_i:.1f} %, of all stall samples {100.0 * sum(x[1] for x in ins if x[2] == mode) / tot_s:.1f} %")
print(f"instructions with that count, in address order ('--' = instructions with another count in between; "
      f"the longest contiguous block has {b - a}):")
print("exec_count  %samples  SASS")
gap = False
for s, smp, e in ins:
    if e == mode:
        if gap:
            print("        --")
        gap = False
        print(f"{e:10d}  {100.0 * smp / tot_s:7.2f}  {s}")
    elif e:
        gap = True
