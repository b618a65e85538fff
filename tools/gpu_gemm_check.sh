timeout 900 python -m pytest tests/test_layer_kernels.py tests/test_gemm_tc.py -x -q > gpurun_out/t1.log 2>&1; echo rc=$? >> gpurun_out/t1.log
python tools/bench_beaver_shapes.py --no-simt > gpurun_out/shapes_new.txt 2>&1
python tools/bench_gemm.py > gpurun_out/gemm4096_st.txt 2>&1
tail -2 gpurun_out/t1.log
