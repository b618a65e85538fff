#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_thin_tc.py -x -q -m gpu > gpurun_out/t_g.log 2>&1; echo rc=$? >> gpurun_out/t_g.log
timeout 600 python bench.py --no-cpu --no-sweep > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
timeout 300 python tools/step_launches.py --arch lenet > gpurun_out/lenet_launch_table.txt 2>&1
tail -3 gpurun_out/t_g.log
