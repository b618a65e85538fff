timeout 300 python tools/micro/softmax_warm.py 2>&1 | tail -3
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/softmax -f python tools/micro/softmax_warm.py > gpurun_out/u_ncu.log 2>&1; tail -1 gpurun_out/u_ncu.log
