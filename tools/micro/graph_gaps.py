"""Idle gaps between consecutive kernels of one graphed LeNet training step
(torch.profiler / CUPTI kernel records of a graph replay): how much of the
step is launch / dependency bubbles rather than kernel time."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2402_02320_b200 import train  # noqa: E402
from paper_2402_02320_b200.preprocessing import DemandCounter  # noqa: E402
from paper_2402_02320_b200.session import SimSession  # noqa: E402

n = 3
dev = torch.device("cuda", 0)
x, y = bench.lenet_data(128)
kx, ky = bench.label_key("share:x"), bench.label_key("share:y")
c = DemandCounter(tuple(range(n)), n)
sd = SimSession(n, c, device=dev)
train.lenet(sd).train_step(sd, sd.share_fixed(x, 64, 23, kx), sd.share_fixed(y, 64, 23, ky), 5)
s = SimSession(n, None, device=dev)
m = train.lenet(s)
xs, ys = s.share_fixed(x, 64, 23, kx), s.share_fixed(y, 64, 23, ky)
g = train.GraphedStep(s, m, xs, ys, 5, c.demands, c.needs_bits, seed0=1)
for i in range(3):
    g.step(10 + i)
torch.cuda.synchronize()
g.dealer.redeal(20)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    g.graph.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
ev.sort(key=lambda e: e.time_range.start)
ks = [(e.time_range.start, e.time_range.end, e.name) for e in ev]
span = ks[-1][1] - ks[0][0]
busy = sum(b - a for a, b, _ in ks)
gaps = [ks[i + 1][0] - ks[i][1] for i in range(len(ks) - 1)]
print(f"{len(ks)} kernels, span {span:.1f} us, kernel time {busy:.1f} us, gaps {sum(max(0, q) for q in gaps):.1f} us "
      f"(median gap {np.median(gaps):.2f} us, max {max(gaps):.1f})")
for (a, b, nm), gp in zip(ks, gaps + [0]):
    print(f"{b - a:8.1f} us  gap {gp:6.2f}  {nm[:70]}")
