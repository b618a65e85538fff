set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python tools/profile_step.py > gpurun_out/step_plain.log 2>&1 && \
ncu --nvtx --nvtx-include "online/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "online/" -k regex:"k_carry_fused|k_bit2a_compose|k_lmo_fused" -c 3 -o gpurun_out/prof_r01 python tools/profile_step.py > gpurun_out/ncu2.log 2>&1
echo done
