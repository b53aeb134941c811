#!/bin/bash
# ncu --set full captures of the kernels besides k_gather_fine: grid build
# (radix passes, permute), the C5 sparse gather, the C3 tracer and the C4
# eye pass.  Each program first runs once without ncu (must exit 0).
set -u
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -f"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-trace --no-render"
timeout 300 $B > gpurun_out/po_bench.json 2>&1; echo "bench rc=$?"
for k in k_radix_downsweep k_permute_packed k_radix_upsweep k_pack_fine k_dense_keys; do
  timeout 600 $NCU -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
C5="python scripts/c5_bench.py --steps 2 --scale ${C5_SCALE:-1}"
timeout 600 $C5 > gpurun_out/po_c5.txt 2>&1; echo "c5 rc=$?"
timeout 900 $NCU -k regex:k_gather_sparse -s 1 -c 1 -o gpurun_out/prof_sparse_c5 $C5 > gpurun_out/ncu_sparse.log 2>&1
echo "sparse rc=$?"
R="python scripts/render_bench.py --steps 2"
timeout 600 $R > gpurun_out/po_render.txt 2>&1; echo "render rc=$?"
timeout 900 $NCU -k regex:k_trace_paths -s 1 -c 1 -o gpurun_out/prof_trace $R > gpurun_out/ncu_trace.log 2>&1
echo "trace rc=$?"
V="python scripts/vcm_profile.py"
timeout 600 $V > gpurun_out/po_vcm.txt 2>&1; echo "vcm rc=$?"
timeout 900 $NCU -k regex:k_eye_bidir -s 2 -c 1 -o gpurun_out/prof_eye_bidir $V > gpurun_out/ncu_eye.log 2>&1
echo "eye rc=$?"
for f in gpurun_out/prof_*.ncu-rep; do python scripts/ncu_summary.py $f; done > gpurun_out/others_summary.txt 2>&1
