set -u
OUT=gpurun_out/profg
mkdir -p $OUT
python tools/bench_beaver_shapes.py --no-simt --only 8192,500,50 --reps 3 > $OUT/plain.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_limbs_tc|k_beaver_limbs" --launch-skip 0 --launch-count 4 -o $OUT/g1 python tools/bench_beaver_shapes.py --no-simt --only 8192,500,50 --reps 1 > $OUT/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_limbs_tc" --launch-count 2 -o $OUT/g2 python tools/bench_beaver_shapes.py --no-simt --only 128,800,500 --reps 1 > $OUT/ncu2.log 2>&1
for r in g1 g2; do
ncu -i $OUT/$r.ncu-rep --page details --csv > $OUT/${r}_details.csv 2>/dev/null
ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>/dev/null
ncu -i $OUT/$r.ncu-rep --page source --csv --print-source sass > $OUT/${r}_sass.csv 2>/dev/null
done
ls -la $OUT
