timeout 300 python -m pytest -q -x tests/test_thin_tc.py > gpurun_out/u_tests.log 2>&1; echo rc=$? >> gpurun_out/u_tests.log; tail -2 gpurun_out/u_tests.log
grep -q "rc=0" gpurun_out/u_tests.log || exit 1
for d in 0 2 7; do echo "dbg $d: $(MPX_THIN_DBG=$d timeout 120 python tools/micro/thin_tc.py --only-thin 2>&1 | tail -1)"; done
