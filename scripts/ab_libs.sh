#!/bin/bash
# A/B of library variants built into build/lib_<name>.so (bench line, C2)
for n in "$@"; do
  L=""; [ "$n" != base ] && L="FPPM_GPU_LIB=build/lib_$n.so"
  env $L timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-trace --no-render --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); r=l['roofline']; print('$n', 'ms/step %.3f gather %.3f frac %.3f' % (l['ms_per_step'], r['avg_launch_ms'], r['frac']))"
done
