export MPX_LONG_DBG=7
timeout 300 ncu --set full --clock-control none -k regex:k_beaver_tc_long -c 1 -o gpurun_out/long_dbg7 -f python tools/micro/long_tc.py --reps 1 > gpurun_out/p_ncu.log 2>&1; tail -1 gpurun_out/p_ncu.log
