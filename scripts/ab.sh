#!/bin/bash
# A/B quick bench of kernel variants (no e2e / cpu baseline)
mkdir -p gpurun_out
Q="--no-e2e --no-cpu-baseline --steps 5 --warmup 3"
summ='import json,sys; d=json.loads(sys.stdin.read().strip().split("\n")[-1]); print(sys.argv[1], round(d["value"]/1e9,3), "Gq/s", round(d["ms_per_step"],3), "ms/step gather", round(d["roofline"]["avg_launch_ms"],3), "frac", round(d["roofline"]["frac"],4))'
for v in ${VARIANTS:-fine tile}; do
  timeout 300 python bench.py $Q --kernel $v ${BENCH_ARGS:-} 2>/dev/null | python -c "$summ" $v
done
if [ -f build/minb1/libfppm_gpu.so ]; then
  FPPM_GPU_LIB=build/minb1/libfppm_gpu.so timeout 300 python bench.py $Q --kernel tile ${BENCH_ARGS:-} 2>/dev/null | python -c "$summ" tile-minb1
fi
