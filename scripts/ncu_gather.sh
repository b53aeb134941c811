#!/bin/bash
# ncu --set full capture of the top gather kernel (plain run first; ncu only if it exits 0)
set -u
mkdir -p gpurun_out
KREGEX=${KREGEX:-k_gather}
TAG=${TAG:-gather}
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-}"
timeout 600 $CMD > gpurun_out/ncu_plain_$TAG.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${SKIP:-3} -c 1 \
   -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?"
