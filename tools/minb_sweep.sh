for tag in A B C; do
  export MPX_LIB=paper_2402_02320_b200/libmpx_$tag.so
  for n in 3 4; do echo "$tag n=$n $(python tools/bench_fused.py --parties $n --elems 4194304 --kinds reciprocal,exp,log,relu 2>&1 | tail -1)"; done
  echo "$tag lenet $(python tools/bench_train.py --graph --steps 5 2>&1 | tail -1)"
done
