#!/bin/bash
# per-kernel launch list of one bench step (run plain first; ncu only if it exits 0)
mkdir -p gpurun_out
CMD="python bench.py --steps ${STEPS:-1} --warmup ${WARMUP:-3} --no-e2e --no-cpu-baseline --no-trace --no-render ${BENCH_ARGS:-}"
timeout 600 $CMD > gpurun_out/launch_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > /dev/null 2>&1
echo "rc=$?"
python scripts/launch_table.py gpurun_out/launches.csv ${SKIP_ITERS:-3} ${PAT:-k_gather}
