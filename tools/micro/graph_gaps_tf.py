"""Per-kernel table (CUPTI records of one graph replay) of the 18.9M Transformer
secure inference (seq 128, n parties simulated): python tools/micro/graph_gaps_tf.py [n]"""
import collections, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200.preprocessing import DemandCounter  # noqa: E402
from paper_2402_02320_b200.session import SimSession  # noqa: E402
from paper_2402_02320_b200.transformer import GraphedInference, Transformer  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda", 0)
x = np.random.default_rng(3).normal(0, 1, (128, 512))
c = DemandCounter(tuple(range(n)), n)
sd = SimSession(n, c, device=dev)
Transformer(sd).forward(sd, sd.share_fixed(x, 64, 14, [5, 5]))
s = SimSession(n, None, device=dev)
m = Transformer(s)
g = GraphedInference(s, m, s.share_fixed(x, 64, 14, [5, 5]), c.demands, c.needs_bits, seed0=90)
for i in range(3):
    g.run(91 + i)
torch.cuda.synchronize()
g.dealer.redeal(95)
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
for k, (t, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{t:9.1f} us {cnt:4d}  {k}")
