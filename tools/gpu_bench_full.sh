# full default bench (driver's command) + timing log
mkdir -p gpurun_out
start=$(date +%s)
timeout 1700 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$? >> gpurun_out/bench_full.err
echo "elapsed $(( $(date +%s) - start )) s" >> gpurun_out/bench_full.err
tail -3 gpurun_out/bench_full.err
