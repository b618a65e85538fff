#!/bin/bash
set -u
mkdir -p gpurun_out
python tools/micro/thin_tc.py > gpurun_out/thin_tc.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_beaver_tc_thin -c 1 -o gpurun_out/thin_tc python tools/micro/thin_tc.py --reps 1 --only-thin > gpurun_out/ncu_thin.log 2>&1
ncu -i gpurun_out/thin_tc.ncu-rep --page source --csv --print-source sass > gpurun_out/thin_tc_source.csv 2>/dev/null
ncu -i gpurun_out/thin_tc.ncu-rep --page details --csv > gpurun_out/thin_tc_details.csv 2>/dev/null
cat gpurun_out/thin_tc.txt
