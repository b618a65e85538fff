#!/bin/bash
# Round-2 first check: smoke, all gpu tests, default bench, reference arm.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
SECONDS=0; timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo rc=$? secs=$SECONDS >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$? >> gpurun_out/bench_ref.err
tail -3 gpurun_out/gpu_tests.log; head -c 600 gpurun_out/bench.json; echo; head -c 400 gpurun_out/bench_ref.json
