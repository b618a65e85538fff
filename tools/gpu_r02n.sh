# long-K tcgen05 Beaver product: unit parity, training parity, step table, quick bench
timeout 600 python -m pytest -q -x tests/test_long_tc.py > gpurun_out/n_tests.log 2>&1; echo rc=$? >> gpurun_out/n_tests.log
tail -15 gpurun_out/n_tests.log
timeout 900 python -m pytest -q -x tests/test_train.py tests/test_gpu_parity.py > gpurun_out/n_tests2.log 2>&1; echo rc=$? >> gpurun_out/n_tests2.log
tail -3 gpurun_out/n_tests2.log
timeout 300 python tools/micro/graph_gaps.py > gpurun_out/n_gaps.txt 2>&1; grep -i "kernels, span\|tc_long\|gemm_sim" gpurun_out/n_gaps.txt | head
timeout 600 python bench.py --no-cpu --no-sweep --steps 20 > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err
python -c "import json;d=json.load(open('gpurun_out/n_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'])"
