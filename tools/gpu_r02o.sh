timeout 120 python -m pytest -q -x tests/test_long_tc.py > gpurun_out/o_tests.log 2>&1; echo rc=$? >> gpurun_out/o_tests.log
tail -3 gpurun_out/o_tests.log
grep -q "rc=0" gpurun_out/o_tests.log || exit 1
timeout 120 python tools/micro/long_tc.py
timeout 300 ncu --set full --clock-control none -k regex:k_beaver_tc_long -c 1 -o gpurun_out/long_tc -f python tools/micro/long_tc.py --reps 1 > gpurun_out/o_ncu.log 2>&1; tail -1 gpurun_out/o_ncu.log
timeout 120 python tools/micro/graph_gaps.py > gpurun_out/o_gaps.txt 2>&1; grep -i "kernels, span\|tc_long\|long_reduce\|gemm_sim" gpurun_out/o_gaps.txt | head
