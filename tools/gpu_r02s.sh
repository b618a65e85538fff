timeout 300 python tools/micro/fc_shapes.py
FC_SWEEP=1 timeout 300 python tools/micro/fc_shapes.py 2>&1 | grep cfg
timeout 900 python -m pytest -q -x tests/test_train.py tests/test_gpu_parity.py tests/test_transformer.py > gpurun_out/s_tests.log 2>&1; echo rc=$? >> gpurun_out/s_tests.log; tail -2 gpurun_out/s_tests.log
timeout 300 python tools/micro/graph_gaps.py > gpurun_out/s_gaps.txt 2>&1; grep -i "kernels, span\|gemm_sim" gpurun_out/s_gaps.txt | head
