#!/bin/bash
# ncu --set full of the fine gather on the fixed iteration-1 state, default lib + $LIBS
mkdir -p gpurun_out
for lib in default ${LIBS}; do
  if [ "$lib" = default ]; then unset FPPM_GPU_LIB; else export FPPM_GPU_LIB=build/$lib/libfppm_gpu.so; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather_fine -s 2 -c 1 \
     -o gpurun_out/ab_$lib -f python scripts/kexp.py > gpurun_out/ncu_ab_$lib.log 2>&1
  echo "$lib rc=$?"
done
