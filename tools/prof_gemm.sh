set -u
OUT=gpurun_out/profg
mkdir -p $OUT
SHAPE=${1:-8192,50,500}
python tools/bench_beaver_shapes.py --no-simt --only $SHAPE --reps 3 > $OUT/plain.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_limbs_tc" --launch-skip 2 --launch-count 1 -o $OUT/g1 python tools/bench_beaver_shapes.py --no-simt --only $SHAPE --reps 1 > $OUT/ncu1.log 2>&1
ncu -i $OUT/g1.ncu-rep --page details --csv > $OUT/g1_details.csv 2>/dev/null
ncu -i $OUT/g1.ncu-rep --page raw --csv > $OUT/g1_raw.csv 2>/dev/null
ncu -i $OUT/g1.ncu-rep --page source --csv --print-source sass > $OUT/g1_sass.csv 2>/dev/null
rm -f $OUT/g1.ncu-rep
