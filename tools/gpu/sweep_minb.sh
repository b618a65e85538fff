#!/bin/bash
# fused Reciprocal / Exp / Log register-cap variants (libmpx_<tag>.so built by tools/build_variant.py)
for v in "" _ldb8 _log10 _log12; do
  if [ -n "$v" ]; then export MPX_LIB=paper_2402_02320_b200/libmpx$v.so; else unset MPX_LIB; fi
  echo "lib$v n2 $(python tools/bench_fused.py --parties 2 --kinds reciprocal,exp,log 2>&1 | tail -1)" >> gpurun_out/sweep_minb.txt
done
unset MPX_LIB
bash tools/gpu/prof_lenet_gemm.sh
