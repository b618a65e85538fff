# quick GPU check: full gpu tests + default bench (no CPU arms / sweep)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu --no-sweep > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python tools/step_launches.py --arch lenet > gpurun_out/lenet_launch_table.txt 2>&1
tail -2 gpurun_out/gpu_tests.log; python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['value'],d['ms_per_step'],d['roofline']['kernel'],d['roofline']['frac'])"
tail -1 gpurun_out/lenet_launch_table.txt
python tools/step_launches.py --arch transformer --parties 2 --summary > gpurun_out/tf_table.txt 2>&1; tail -2 gpurun_out/tf_table.txt
