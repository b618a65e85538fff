# tiled trunc_expand_rows check: training parity + LeNet step table + quick bench
timeout 900 python -m pytest -q -x tests/test_train.py tests/test_layer_kernels.py tests/test_party_layer.py > gpurun_out/m_tests.log 2>&1; echo rc=$? >> gpurun_out/m_tests.log
tail -3 gpurun_out/m_tests.log
timeout 300 python tools/micro/graph_gaps.py > gpurun_out/m_gaps.txt 2>&1; grep -i "trunc_expand\|step\|total" gpurun_out/m_gaps.txt | head
timeout 600 python bench.py --no-cpu --no-sweep --steps 20 > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
python -c "import json;d=json.load(open('gpurun_out/m_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'])"
