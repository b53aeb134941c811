#!/bin/bash
# A/B: default library vs alternative builds under build/*/libfppm_gpu.so
summ='import json,sys; d=json.load(open(sys.argv[2])); r=d["roofline"]; print(sys.argv[1], "kernel", round(sum(r["launch_ms"])/len(r["launch_ms"]),3), "step", round(d["ms_per_step"],3), "Gq/s", round(d["value"]/1e9,2))'
for lib in default ${LIBS}; do
  if [ "$lib" = default ]; then unset FPPM_GPU_LIB; else export FPPM_GPU_LIB=build/$lib/libfppm_gpu.so; fi
  timeout 300 python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-trace --no-render > gpurun_out/ab_$lib.json 2>/dev/null && python -c "$summ" $lib gpurun_out/ab_$lib.json
done
