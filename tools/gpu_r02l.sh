#!/bin/bash
# ncu full captures: conv2-forward mask+limb kernel, fused Log (n = 2, 2^22), fused Reciprocal n = 8 (L4G2)
set -u
mkdir -p gpurun_out/prof
O=gpurun_out/prof
timeout 300 python -m pytest -q tests/test_thin_tc.py tests/test_gemm_tc.py tests/test_layer_kernels.py tests/test_fused_ops.py > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mask_limbs2 -c 1 -o $O/mask_conv2 python tools/micro/gemm_split_shapes.py --only 8192,500,50 --reps 1 --no-check > $O/ncu1.log 2>&1
ncu -i $O/mask_conv2.ncu-rep --page details --csv > $O/mask_conv2_details.csv 2>/dev/null
ncu -i $O/mask_conv2.ncu-rep --page source --csv --print-source sass > $O/mask_conv2_source.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_log_fused -c 1 -o $O/log_n2 python tools/bench_fused.py --kinds log --elems 4194304 --reps 1 > $O/ncu2.log 2>&1
ncu -i $O/log_n2.ncu-rep --page details --csv > $O/log_n2_details.csv 2>/dev/null
ncu -i $O/log_n2.ncu-rep --page source --csv --print-source sass > $O/log_n2_source.csv 2>/dev/null
rm -f $O/*.ncu-rep
ls -la $O
