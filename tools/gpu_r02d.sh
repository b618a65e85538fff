#!/bin/bash
# split-GEMM knob sweep at the LeNet shapes (timing experiments; DBG runs give wrong results)
set -u
mkdir -p gpurun_out
O=gpurun_out/gemm_knobs.txt; : > $O
for st in 1 0; do for ks in 0 1 2 4; do
  echo "== STAGED=$st KSPLIT=$ks" >> $O
  if [ $ks = 0 ]; then MPX_TC_STAGED=$st timeout 200 python tools/micro/gemm_split_shapes.py --no-check >> $O 2>&1
  else MPX_TC_STAGED=$st MPX_TC_KSPLIT=$ks timeout 200 python tools/micro/gemm_split_shapes.py --no-check >> $O 2>&1; fi
done; done
for dbg in 4 2 8 16 6; do
  echo "== DBG=$dbg" >> $O
  MPX_TC_DBG=$dbg timeout 200 python tools/micro/gemm_split_shapes.py --no-check >> $O 2>&1
done
echo done
