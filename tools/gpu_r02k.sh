#!/bin/bash
set -u
mkdir -p gpurun_out
SECONDS=0; timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? secs=$SECONDS >> gpurun_out/gpu_tests.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep"
$CMD > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
python tools/launch_steps.py gpurun_out/bench_launches.csv > gpurun_out/step_table.txt 2>&1
tail -3 gpurun_out/gpu_tests.log
