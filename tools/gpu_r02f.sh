#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_thin_tc.py tests/test_dealer_fused.py tests/test_train.py tests/test_bench_configs.py -x -q -m gpu -k "not sweep and not freivalds and not transformer" > gpurun_out/t_f.log 2>&1; echo rc=$? >> gpurun_out/t_f.log
timeout 300 python tools/micro/dealer_profile.py > gpurun_out/dealer_profile_fused.txt 2>&1
timeout 600 python bench.py --no-cpu --no-sweep > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
MPX_THIN_TC=0 timeout 600 python bench.py --no-cpu --no-sweep > gpurun_out/bench_quick_nothin.json 2>> gpurun_out/bench_quick.err
tail -3 gpurun_out/t_f.log
