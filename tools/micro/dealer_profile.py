"""Per-kernel breakdown of one LeNet re-deal (n = 3, batch 128), the Philox
ALU ceiling (k_philox_elems on a 1 GiB buffer), and the dealer graph time."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
from paper_2402_02320_b200 import _lib, kernels as K, train
from paper_2402_02320_b200.preprocessing import DemandCounter, DealerGraph, device_store
from paper_2402_02320_b200.session import SimSession

n = 3
x, y = bench.lenet_data(128)
c = DemandCounter(tuple(range(n)), n)
sd = SimSession(n, c)
train.lenet(sd).train_step(sd, sd.share_fixed(x, 64, 23, [1, 1]), sd.share_fixed(y, 64, 23, [1, 2]), 5)
for k, v in sorted(c.demands.items(), key=lambda kv: kv[0].name()):
    print(f"  {k.name():28s} {v:>12d}")
st = device_store(1, n, c.demands, needs_bits=c.needs_bits)
torch.cuda.synchronize()
_lib.profile_begin()
device_store(2, n, c.demands, needs_bits=c.needs_bits, into=st)
torch.cuda.synchronize()
prof = _lib.profile_end()
agg = {}
for nm, a, e0, e1 in prof:
    d = agg.setdefault(nm, [0.0, 0])
    d[0] += e0.elapsed_time(e1)
    d[1] += 1
tot = sum(v[0] for v in agg.values())
print(f"eager re-deal: {tot:.3f} ms in {sum(v[1] for v in agg.values())} launches")
for nm, (ms, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {ms:8.3f} ms {cnt:4d}  {nm}")
g = DealerGraph(st, c.demands, c.needs_bits, 3)
ts = []
for i in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.redeal(10 + i); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("graph re-deal ms", [round(t, 3) for t in ts])
import bench
from paper_2402_02320_b200.preprocessing import stream_blocks
blocks = stream_blocks(c.demands, n, c.needs_bits)
peak = bench.philox_ceiling_gblocks(torch)
ms = min(ts)
print(f"philox ceiling (mpx_philox_probe): {peak:.1f} G blocks/s; re-deal: {blocks / 1e6:.1f} M blocks in {ms:.3f} ms "
      f"= {blocks / ms / 1e6:.1f} G blocks/s = {blocks / ms / 1e6 / peak:.2f} of the ALU ceiling")
