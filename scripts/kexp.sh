#!/bin/bash
for lib in default ${LIBS}; do
  if [ "$lib" = default ]; then unset FPPM_GPU_LIB; else export FPPM_GPU_LIB=build/$lib/libfppm_gpu.so; fi
  timeout 300 python scripts/kexp.py
done
