timeout 300 python tools/micro/softmax_warm.py 2>&1 | tail -1
timeout 900 python -m pytest -q -x tests/test_train.py tests/test_gpu_parity.py tests/test_fused_ops.py > gpurun_out/w_tests.log 2>&1; echo rc=$? >> gpurun_out/w_tests.log; tail -2 gpurun_out/w_tests.log
timeout 300 python tools/micro/graph_gaps.py > gpurun_out/w_gaps.txt 2>&1; grep -i "kernels, span\|softmax" gpurun_out/w_gaps.txt | head
