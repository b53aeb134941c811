#!/usr/bin/env python
"""Print the SASS of one kernel (nvdisasm -g output) restricted to source
lines [lo, hi] of a file, with the line number of each instruction."""
import re, sys
path, func, fname, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
cur = None; line = None; inside = False; n = 0
for l in open(path):
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m:
        inside = func in m.group(1)
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = int(m.group(2)) if fname in m.group(1) else None
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?);', l)
    if m and line is not None and lo <= line <= hi:
        print(f"{m.group(1)} L{line:5d}  {m.group(2)}")
        n += 1
    elif re.match(r'\.L_x_\d+:', l.strip()) and inside:
        print(l.strip())
print("count", n, file=sys.stderr)
