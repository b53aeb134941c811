#!/bin/bash
# bench line (counters) + ncu --set full of the fine gather kernel
mkdir -p gpurun_out
TAG=${TAG:-fine}
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-trace --no-render ${BENCH_ARGS:-}"
timeout 600 $CMD > gpurun_out/ncu_plain_$TAG.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_gather_ring} -s ${SKIP:-3} -c 1 \
   -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_plain_$TAG.json | cut -c 1-3000
