timeout 900 python -m pytest -q -x tests/test_thin_tc.py tests/test_train.py tests/test_gpu_parity.py tests/test_bench_configs.py > gpurun_out/v_tests.log 2>&1; echo rc=$? >> gpurun_out/v_tests.log; tail -2 gpurun_out/v_tests.log
timeout 300 python tools/micro/graph_gaps.py > gpurun_out/v_gaps.txt 2>&1; grep -i "kernels, span\|tc_thin" gpurun_out/v_gaps.txt | head
