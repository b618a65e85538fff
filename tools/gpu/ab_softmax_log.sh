python -m pytest tests/test_fused_ops.py tests/test_train.py tests/test_bench_configs.py tests/test_layer_kernels.py -q -m gpu -x -k "softmax or lenet or maxcut or beaver_gemm_sim" > gpurun_out/t12.log 2>&1
python tools/micro/softmax_warm.py >> gpurun_out/t12.log 2>&1
MPX_SOFTMAX_SPLIT3=0 python tools/micro/softmax_warm.py >> gpurun_out/t12.log 2>&1
python tools/bench_train.py --graph --steps 5 >> gpurun_out/t12.log 2>&1
for v in "" _log4 _log5 _log8; do
  if [ -n "$v" ]; then export MPX_LIB=paper_2402_02320_b200/libmpx$v.so; fi
  echo "lib$v n2 $(python tools/bench_fused.py --parties 2 --kinds log 2>&1 | tail -1)" >> gpurun_out/t12.log
done
