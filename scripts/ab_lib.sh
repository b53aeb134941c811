mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -rf -k "regions or edge" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
FPPM_GPU_LIB=build/libfppm_gpu_old.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_old_$i.json 2>gpurun_out/ab_old.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_new_$i.json 2>gpurun_out/ab_new.err
done
tail -5 gpurun_out/pytest_gpu.log
for f in gpurun_out/ab_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value']/1e9, d['roofline']['avg_launch_ms'], d['ms_per_step'])"; done
