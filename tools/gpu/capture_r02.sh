#!/bin/bash
# Round-2 profile capture on one B200: launch list of the bench step and full
# ncu sections of the hot kernels. Each ncu command runs after the same command
# exited 0 without ncu. Output: gpurun_out/prof2/ (raw CSVs, no .ncu-rep).
set -u
O=gpurun_out/prof2
mkdir -p $O
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep"
$CMD > $O/bench_plain.json 2> $O/bench_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv $CMD > $O/ncu_launches.log 2>&1
python tools/launch_steps.py $O/bench_launches.csv > $O/step_table.txt 2>&1
cap() {  # name regex command...
  local name=$1 rx=$2; shift 2
  "$@" > $O/${name}_plain.log 2>&1 || { echo "plain run failed: $name" >> $O/errors.txt; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -o $O/$name "$@" > $O/ncu_$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page raw --csv --metrics $M > $O/${name}_raw.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  rm -f $O/$name.ncu-rep
}
cap lenet_split_gemm k_gemm_limbs_tc_pers python tools/micro/gemm_split_shapes.py --reps 1 --no-check
cap lenet_mask k_mask_limbs2 python tools/micro/gemm_split_shapes.py --reps 1 --no-check
cap gemm4096 k_gemm_limbs_tc_pers python tools/micro/gemm_split_shapes.py --only 4096,4096,4096 --parties 2 --reps 1 --no-check
cap thin_conv1 k_beaver_tc_thin python tools/micro/thin_tc.py --reps 1 --only-thin
cap recip_fused k_reciprocal_fused python tools/bench_fused.py --kinds reciprocal --elems 4194304 --reps 1
cap deal_bintriple k_deal_bintriple python tools/micro/deal_bintriple.py
ls -la $O
