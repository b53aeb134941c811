#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, default bench + reference arm,
# C1 / C5 bench lines, launch list + ncu of the C2 gather, C5 launch list + ncu of
# the 3D gather and its prep kernel.
set -u
mkdir -p gpurun_out
bash scripts/round_profile.sh
timeout 600 python bench.py --workload c1 --no-trace --no-render > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --workload c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
bash scripts/c5_profile.sh
timeout 900 ncu --set full --clock-control none -f -k regex:k_prep_3d -s 1 -c 1 -o gpurun_out/prof_prep3d python scripts/c5_bench.py --steps 2 > gpurun_out/ncu_prep3d.log 2>&1; echo "prep ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_prep3d.ncu-rep > gpurun_out/prof_prep3d_summary.txt 2>&1
python scripts/step_profile.py > gpurun_out/step_profile.txt 2>&1
