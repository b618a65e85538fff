# Log fused kernel: timing + one ncu --set full capture at 2^22, n = 2
timeout 300 python tools/bench_fused.py --kinds log --elems 4194304 2>&1 | tail -3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_log_fused -c 1 -o gpurun_out/log_fused -f python tools/bench_fused.py --kinds log --elems 4194304 --reps 1 > gpurun_out/r_ncu.log 2>&1; tail -1 gpurun_out/r_ncu.log
