#!/bin/bash
# Step anatomy: eager launch table, dealer breakdown, ncu launch list of the graphed bench step.
set -u
mkdir -p gpurun_out
timeout 300 python tools/step_launches.py --arch lenet > gpurun_out/lenet_launch_table.txt 2>&1
timeout 300 python tools/micro/dealer_profile.py > gpurun_out/dealer_profile.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep"
$CMD > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo done
