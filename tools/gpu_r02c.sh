#!/bin/bash
set -u
mkdir -p gpurun_out
./tools/micro/philox_bench > gpurun_out/philox_bench.txt 2>&1
timeout 300 python tools/micro/gemm_split_shapes.py > gpurun_out/gemm_split_shapes.txt 2>&1
for s in 1 2 3 4; do MPX_TC_KSPLIT=$s timeout 120 python tools/micro/gemm_split_shapes.py --only 8192,500,50 --no-check; done > gpurun_out/gemm_conv2_splits.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_limbs_tc_pers -c 1 \
   -o gpurun_out/conv2_fwd_gemm python tools/micro/gemm_split_shapes.py --only 8192,500,50 --reps 1 --no-check > gpurun_out/ncu_conv2.log 2>&1
ncu -i gpurun_out/conv2_fwd_gemm.ncu-rep --page raw --csv > gpurun_out/conv2_fwd_gemm_raw.csv 2>/dev/null
ncu -i gpurun_out/conv2_fwd_gemm.ncu-rep --page source --csv --print-source sass > gpurun_out/conv2_fwd_gemm_source.csv 2>/dev/null
ncu -i gpurun_out/conv2_fwd_gemm.ncu-rep --page details --csv > gpurun_out/conv2_fwd_gemm_details.csv 2>/dev/null
echo done
