#!/bin/bash
# every GPU test + the C5 / C3 / C4 timings
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -rf > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/fc_pytest.log
timeout 600 python scripts/c5_bench.py --steps 3 > gpurun_out/fc_c5.txt 2>&1; echo "c5 rc=$?"; cat gpurun_out/fc_c5.txt | tail -3
timeout 600 python scripts/render_bench.py --steps 3 > gpurun_out/fc_c3.txt 2>&1; echo "c3 rc=$?"; tail -2 gpurun_out/fc_c3.txt
timeout 600 python scripts/vcm_profile.py > gpurun_out/fc_c4.txt 2>&1; echo "c4 rc=$?"; grep -v Warn gpurun_out/fc_c4.txt | head -8
