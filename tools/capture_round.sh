#!/bin/bash
# Round-end profile capture on one B200 (through gpurun). Each ncu command runs
# only after the same command exited 0 without ncu. Output: gpurun_out/prof/.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep"
$CMD > $OUT/bench_plain.json 2> $OUT/bench_plain.err || exit 1
# launch list of the bench command itself (per-launch times cold/serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bench_launches.csv $CMD \
    > $OUT/ncu_bench_launches.log 2>&1
python tools/bench_train.py --graph --steps 2 > $OUT/bench_train.json 2>&1 || exit 1
# full sections for the step's tcgen05 GEMMs and fused Beaver-operand kernels
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_limbs_tc_pers|k_mask_limbs|k_beaver_gemm_sim" \
    --launch-skip 30 --launch-count 20 -o $OUT/lenet_gemm_full python tools/bench_train.py --graph --steps 1 \
    > $OUT/ncu_lenet_gemm_full.log 2>&1
ncu -i $OUT/lenet_gemm_full.ncu-rep --page details --csv > $OUT/lenet_gemm_full_details.csv 2>/dev/null
ncu -i $OUT/lenet_gemm_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,lts__t_sector_hit_rate.pct > $OUT/lenet_gemm_full_raw.csv 2>/dev/null
rm -f $OUT/lenet_gemm_full.ncu-rep
ls -la $OUT
