#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
SECONDS=0; timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? secs=$SECONDS >> gpurun_out/gpu_tests.log
timeout 300 python tools/micro/dealer_profile.py > gpurun_out/dealer_profile.txt 2>&1
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? secs=$SECONDS >> gpurun_out/bench.err
tail -2 gpurun_out/gpu_tests.log; head -c 400 gpurun_out/bench.json
