timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 900 python -c "
import sys, json, torch; sys.argv=['bench.py']; import bench
import paper_2402_02320_b200 as G
from bench import DistGroup, party_scaling
import torch.distributed as dist
g = DistGroup(torch, dist)
print(json.dumps(party_scaling(torch, G, torch.device('cuda',0), g, ns=(4, 8))))
" > gpurun_out/party.json 2> gpurun_out/party.err; tail -c 1500 gpurun_out/party.json; tail -3 gpurun_out/party.err
