#!/bin/bash
# Full round evidence: GPU tests, default bench (value + e2e + cpu baseline),
# reference arm, launch list, one ncu --set full capture of the gather kernel.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
STEPS=${STEPS:-2} bash scripts/launches.sh > gpurun_out/launches.txt 2>&1; echo "launches rc=$?"
bash scripts/ncu_fine.sh > gpurun_out/ncu_fine.txt 2>&1; echo "ncu rc=$?"
# C3 full-iteration launch list (light phase + eye pass + grid + sparse gather + film)
timeout 600 python scripts/render_bench.py --steps 2 > gpurun_out/render_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/render_launches.csv python scripts/render_bench.py --steps 2 > /dev/null 2>&1; echo "render launches rc=$?"
# C4 full VCM+ iteration launch list
timeout 600 python scripts/vcm_profile.py > gpurun_out/vcm_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vcm_launches.csv python scripts/vcm_profile.py > /dev/null 2>&1; echo "vcm launches rc=$?"
