#!/bin/bash
# Round profile capture on one B200 (run through gpurun). Each ncu command
# runs only after the same command exited 0 without ncu. Reports are reduced
# to CSV on the box (gpurun copies back <= 64 MiB).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
reduce() {  # $1 = report basename
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1_details.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio > $OUT/$1_raw.csv 2>/dev/null
  rm -f $OUT/$1.ncu-rep
}
if [ "${1:-all}" = "all" ] || [ "$1" = "lenet" ]; then
python tools/bench_train.py --graph --steps 3 > $OUT/bench_train.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/lenet_launches.csv \
    python tools/bench_train.py --graph --steps 1 > $OUT/ncu_launches.log 2>&1
ncu --set full --clock-control none \
    -k regex:"k_gemm_limbs_tc|k_mask_limbs|k_relu_fused|k_beaver_gemm|k_mask_sub|k_trunc_fused|k_beaver_limbs_a" \
    --launch-skip 6 --launch-count 40 -o $OUT/lenet_full python tools/bench_train.py --graph --steps 1 \
    > $OUT/ncu_lenet_full.log 2>&1
reduce lenet_full
fi
if [ "${1:-all}" = "all" ] || [ "$1" = "nonlinear" ]; then
python tools/bench_fused.py --kinds reciprocal,exp,log > $OUT/bench_fused.json 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_(reciprocal|exp|log)_fused" \
    -o $OUT/nonlinear_full python tools/bench_fused.py --kinds reciprocal,exp,log --reps 1 \
    > $OUT/ncu_nonlinear.log 2>&1
reduce nonlinear_full
fi
if [ "${1:-all}" = "all" ] || [ "$1" = "gemm" ]; then
python tools/bench_gemm.py > $OUT/bench_gemm.json 2>&1 || exit 1
ncu --set full --clock-control none -k regex:k_gemm_limbs_tc --launch-skip 3 --launch-count 1 \
    -o $OUT/gemm4096_full python tools/bench_gemm.py --iters 1 > $OUT/ncu_gemm.log 2>&1
reduce gemm4096_full
fi
if [ "${1:-all}" = "all" ] || [ "$1" = "split8" ]; then
# n = 8 sim-mode fused kernels with the party split (2^22 elements)
python tools/bench_fused.py --parties 8 --elems 4194304 --kinds reciprocal,exp,log,relu > $OUT/bench_fused8.json 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_(reciprocal|exp|log|relu)_fused" \
    -o $OUT/split8_full python tools/bench_fused.py --parties 8 --elems 4194304 --kinds reciprocal,exp,log,relu --reps 1 \
    > $OUT/ncu_split8.log 2>&1
reduce split8_full
fi
echo done
