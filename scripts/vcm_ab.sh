#!/bin/bash
# A/B of library variants on the C4 VCM+ iteration (per-kernel profile)
for lib in default ${LIBS}; do
  if [ "$lib" = default ]; then unset FPPM_GPU_LIB; else export FPPM_GPU_LIB=build/$lib/libfppm_gpu.so; fi
  echo "== $lib"; timeout 300 python scripts/vcm_profile.py 2>&1 | grep -E "per iteration|k_eye_bidir"
done
