#!/bin/bash
# parity of the default (fine) path + the bench line without the side legs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_fullsize.py tests/test_gpu_regions.py tests/test_gpu_edge.py -x -q ${PYTEST_ARGS:-} > gpurun_out/qc_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/qc_pytest.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-trace --no-render ${BENCH_ARGS:-} > gpurun_out/qc_bench.json 2> gpurun_out/qc_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open('gpurun_out/qc_bench.json').read().strip().split('\n')[-1])
r=l['roofline']
print("value %.3g ms/step %.3f gather %.3f ms frac %.3f launches %s" % (l['value'], l['ms_per_step'], r['avg_launch_ms'], r['frac'], l['gpu_launches']))
PY
