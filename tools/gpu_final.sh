#!/bin/bash
# Final round check: smoke, all GPU tests, default bench, reference arm, party-mode bench path (2 threads).
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
SECONDS=0; timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? secs=$SECONDS >> gpurun_out/gpu_tests.log
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc=$? secs=$SECONDS >> gpurun_out/bench.err
SECONDS=0; timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rc=$? secs=$SECONDS >> gpurun_out/bench_ref.err
tail -2 gpurun_out/gpu_tests.log; head -c 300 gpurun_out/bench.json; echo; head -c 300 gpurun_out/bench_ref.json
