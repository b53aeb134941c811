#!/usr/bin/env python
"""Print the innermost SASS loop of a kernel that contains code from source
line L of a file (nvdisasm -g output): the block from the branch target of
the first backward branch that jumps over an instruction of line L."""
import re, sys
path, func, fname, L = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
ins = []; inside = False; line = None; labels = {}
for l in open(path):
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m:
        if inside: break
        inside = func in m.group(1); continue
    if not inside: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: line = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*(\.L_x_\d+):', l)
    if m: labels[m.group(1)] = len(ins); continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if m: ins.append((int(m.group(1), 16), line, m.group(2).strip()))
hit = [k for k, x in enumerate(ins) if x[1] and x[1][0] == fname and x[1][1] == L]
best = None
for k, x in enumerate(ins):
    m = re.search(r'BRA\s+`?\(?(\.L_x_\d+)', x[2])
    if m and m.group(1) in labels:
        t = labels[m.group(1)]
        if t <= k and any(t <= h <= k for h in hit):
            if best is None or k - t < best[1] - best[0]:
                best = (t, k)
t, k = best
for a, ln, txt in ins[t:k + 1]:
    print(f"{a:05x} {ln[1] if ln else '':>5} {txt}")
print(f"loop: {k - t + 1} instructions", file=sys.stderr)
