#!/usr/bin/env python
"""Attribute an ncu SASS source page (csv) to CUDA source lines.

usage: ncu_lines.py SASS_CSV NVDISASM_G_OUT FUNC_SUBSTR [FILE_SUBSTR]

The ncu csv (--page source --csv --print-source sass) lists the kernel's
instructions in address order; nvdisasm -g of the same cubin gives the
source line of each instruction offset.  Prints stall samples, warp
instructions and the top stall reasons per source line, sorted by samples."""
import collections, csv, os, re, sys

csv_path, dis_path, func = sys.argv[1], sys.argv[2], sys.argv[3]
fsub = sys.argv[4] if len(sys.argv) > 4 else ''

line_of = {}
inside = False
cur = None
for l in open(dis_path):
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m:
        if inside:
            break
        inside = func in m.group(1)
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        mi = re.search(r'inlined at "([^"]+)", line (\d+)', l)
        if mi and os.environ.get('OUTER'):  # attribute helpers (nvdisasm -gi) to their call site
            cur = (mi.group(1).split('/')[-1], int(mi.group(2)))
        elif 'inlined at' not in l or os.environ.get('INNER'):
            cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if m:
        line_of[int(m.group(1), 16)] = cur

rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
base = int(data[0][ix['Address']], 16)
stall_cols = [h for h in hdr if h.startswith('stall_') and '(Not Issued)' not in h]
agg = collections.defaultdict(lambda: collections.Counter())
tot_s = tot_i = 0
for r in data:
    off = int(r[ix['Address']], 16) - base
    key = line_of.get(off)
    key = key if key and fsub in key[0] else (key or ('?', 0))
    s = float(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    n = float(r[ix['Instructions Executed']] or 0)
    c = agg[key]
    c['samples'] += s
    c['inst'] += n
    for h in stall_cols:
        v = float(r[ix[h]] or 0)
        if v:
            c[h] += v
    tot_s += s
    tot_i += n
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.4g}")
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]['samples'])[:int(sys.argv[5]) if len(sys.argv) > 5 else 60]:
    top = sorted(((v, h[6:]) for h, v in c.items() if h.startswith('stall_')), reverse=True)[:3]
    tops = ' '.join(f"{h}:{100 * v / max(c['samples'], 1):.0f}%" for v, h in top)
    print(f"{key[0]:>16}:{key[1]:<5} {100 * c['samples'] / tot_s:5.1f}% samp {100 * c['inst'] / tot_i:5.1f}% inst  {tops}")
