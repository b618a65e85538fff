#!/bin/bash
# ncu source-level capture of the LeNet step's tcgen05 GEMMs and mask+limb
# kernels (graph replay after the eager warm-up step).
OUT=gpurun_out/prof_gemm
mkdir -p $OUT
python tools/bench_train.py --graph --steps 1 > $OUT/plain.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_limbs_tc_pers|k_mask_limbs2" \
    --launch-skip 12 --launch-count 4 -o $OUT/lenet_gemm python tools/bench_train.py --graph --steps 1 > $OUT/ncu.log 2>&1
ncu -i $OUT/lenet_gemm.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/lenet_gemm.ncu-rep --page source --csv --print-source sass > $OUT/source.csv 2>/dev/null
ncu -i $OUT/lenet_gemm.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct > $OUT/raw.csv 2>/dev/null
rm -f $OUT/lenet_gemm.ncu-rep
