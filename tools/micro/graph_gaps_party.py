"""Per-kernel table (CUPTI records of one graph replay) of party 0's share of
the one-party-per-GPU LeNet step (LoopbackComm: collectives elided):
python tools/micro/graph_gaps_party.py [n]"""
import collections, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2402_02320_b200 import train  # noqa: E402
from paper_2402_02320_b200.preprocessing import DemandCounter  # noqa: E402
from paper_2402_02320_b200.session import LoopbackComm, PartySession  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
x, y = bench.lenet_data(128)
kx, ky = bench.label_key("share:x"), bench.label_key("share:y")
c = DemandCounter((0,), n)
sd = PartySession(0, n, LoopbackComm(n), c, device=dev)
train.lenet(sd).train_step(sd, sd.share_fixed(x, 64, 23, kx), sd.share_fixed(y, 64, 23, ky), 5)
s = PartySession(0, n, LoopbackComm(n), None, device=dev)
m = train.lenet(s)
g = train.GraphedStep(s, m, s.share_fixed(x, 64, 23, kx), s.share_fixed(y, 64, 23, ky), 5, c.demands, c.needs_bits,
                      seed0=300)
for i in range(3):
    g.step(301 + i)
torch.cuda.synchronize()
g.dealer.redeal(305)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    g.graph.replay()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
ev.sort(key=lambda e: e.time_range.start)
span = ev[-1].time_range.end - ev[0].time_range.start
agg = collections.defaultdict(lambda: [0.0, 0])
for e in ev:
    k = e.name.split("(")[0].replace("void ", "")[:60]
    agg[k][0] += e.time_range.elapsed_us()
    agg[k][1] += 1
busy = sum(v[0] for v in agg.values())
print(f"{len(ev)} kernels, span {span:.1f} us, kernel time {busy:.1f} us")
for k, (t, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{t:9.1f} us {cnt:4d}  {k}")
