#!/bin/bash
# every GPU test + the C5 / C3 / C4 timings
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -rf > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/fc_pytest.log
timeout 600 python scripts/c5_bench.py --steps 3 > gpurun_out/fc_c5.txt 2>&1; echo "c5 rc=$?"; cat gpurun_out/fc_c5.txt | tail -3
timeout 600 python scripts/render_bench.py --steps 3 > gpurun_out/fc_c3.txt 2>&1; echo "c3 rc=$?"; tail -2 gpurun_out/fc_c3.txt
timeout 600 python scripts/vcm_profile.py > gpurun_out/fc_c4.txt 2>&1; echo "c4 rc=$?"; grep -v Warn gpurun_out/fc_c4.txt | head -8
if [ -n "${NCU3D:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:k_gather_3d -s 1 -c 1 -o gpurun_out/prof_3d python scripts/c5_bench.py --steps 2 > gpurun_out/ncu_3d.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_3d.ncu-rep > gpurun_out/prof_3d_summary.txt 2>&1
  ncu -i gpurun_out/prof_3d.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_3d_src.csv 2>/dev/null
fi
