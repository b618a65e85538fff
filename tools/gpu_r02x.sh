for v in "" roll; do
  if [ -n "$v" ]; then export MPX_LIB=$PWD/paper_2402_02320_b200/libmpx_$v.so; else unset MPX_LIB; fi
  echo "== ${v:-default}"
  timeout 300 python tools/bench_fused.py --kinds reciprocal,exp,log,relu 2>&1 | tail -1
  timeout 300 python tools/bench_fused.py --kinds reciprocal,exp,log --parties 3 --elems 4194304 2>&1 | tail -1
  timeout 300 python tools/micro/graph_gaps.py 2>&1 | grep -i "kernels, span\|relu_fused"
done
