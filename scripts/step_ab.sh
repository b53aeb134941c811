#!/bin/bash
# A/B of library variants: warm per-kernel profile of a C2 step
for lib in default ${LIBS}; do
  if [ "$lib" = default ]; then unset FPPM_GPU_LIB; else export FPPM_GPU_LIB=build/$lib/libfppm_gpu.so; fi
  echo "== $lib"; timeout 300 python scripts/step_profile.py 2>&1 | grep -E "per step|${PAT:-finalize}"
done
