#!/bin/bash
# quick loop: fine parity tests + 8-step bench summary
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "${PYTEST_K:-fine or regions or edge}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/b.json 2>gpurun_out/b.err
python -c "import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('kernel ms', r['launch_ms'], 'step', round(d['ms_per_step'],3), 'Gq/s', round(d['value']/1e9,2), 'frac', round(r['frac'],4))"
