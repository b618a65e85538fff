timeout 900 python -m pytest -q -x tests/test_fused_ops.py tests/test_train.py tests/test_gpu_parity.py tests/test_transformer.py > gpurun_out/x_tests.log 2>&1; echo rc=$? >> gpurun_out/x_tests.log; tail -2 gpurun_out/x_tests.log
timeout 300 python tools/micro/graph_gaps.py 2>&1 | grep -i "kernels, span\|relu_fused"
timeout 300 python tools/bench_fused.py --kinds relu --elems 65536 2>&1 | tail -1
