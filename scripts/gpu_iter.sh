#!/bin/bash
# quick GPU iteration: parity tests (selection via PYTEST_K) + A/B bench
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -q -m gpu -rf -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
bash scripts/ab.sh 2>&1 | tee gpurun_out/ab.txt
