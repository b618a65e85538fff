"""Is the fused LeNet softmax (128 x 10, n = 3) DRAM-latency bound? Time it
with cold material (fresh deal) and again with the same material L2-hot
(cursors rewound)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import nn, _lib
from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
from paper_2402_02320_b200.session import SimSession

n = int(os.environ.get("N", 3))
rows, cols = int(os.environ.get("ROWS", 128)), int(os.environ.get("COLS", 10))
x = np.random.default_rng(1).normal(0, 3, (rows, cols))
c = DemandCounter(tuple(range(n)), n)
sd = SimSession(n, c)
nn.softmax_parts(sd, sd.share_fixed(x, 64, 23, [1, 1]))
for trial in range(3):
    st = device_store(5 + trial, n, c.demands, needs_bits=c.needs_bits)
    s = SimSession(n, st)
    xs = s.share_fixed(x, 64, 23, [1, 1])
    big = torch.empty(1 << 28, dtype=torch.uint8, device="cuda"); big.zero_(); del big   # flush L2
    torch.cuda.synchronize()
    res = []
    for rep in range(3):
        st.rewind()
        _lib.profile_begin()
        nn.softmax_parts(s, xs)
        torch.cuda.synchronize()
        prof = _lib.profile_end()
        res.append(sum(a.elapsed_time(b) for nm, _, a, b in prof if "softmax" in nm or "maxtour" in nm) * 1e3)
    print(f"trial {trial}: cold {res[0]:.1f} us, L2-hot {res[1]:.1f} / {res[2]:.1f} us  "
          f"kernels {sorted(set(nm for nm, *_ in prof))}")
