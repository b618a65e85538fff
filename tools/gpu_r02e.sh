#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dealer_fused.py tests/test_gpu_parity.py tests/test_material_io.py tests/test_train.py -x -q -m gpu > gpurun_out/dealer_tests.log 2>&1; echo rc=$? >> gpurun_out/dealer_tests.log
timeout 300 python tools/micro/dealer_profile.py > gpurun_out/dealer_profile_fused.txt 2>&1
MPX_DEALER_LEGACY=1 timeout 300 python tools/micro/dealer_profile.py > gpurun_out/dealer_profile_legacy.txt 2>&1
tail -3 gpurun_out/dealer_tests.log
