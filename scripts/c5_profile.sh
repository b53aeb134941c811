mkdir -p gpurun_out
timeout 900 python scripts/c5_bench.py --steps 3 > gpurun_out/c5_plain.txt 2>&1; echo "c5 rc=$?"; tail -3 gpurun_out/c5_plain.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python scripts/c5_bench.py --steps 2 > /dev/null 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -f -k regex:k_gather_3d -s 1 -c 1 -o gpurun_out/prof_3d python scripts/c5_bench.py --steps 2 > gpurun_out/ncu_3d.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_3d.ncu-rep > gpurun_out/prof_3d_summary.txt 2>&1
ncu -i gpurun_out/prof_3d.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_3d_src.csv 2>/dev/null
