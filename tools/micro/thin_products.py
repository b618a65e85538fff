"""LeNet conv1's two Beaver products (n = 3, batch 128) in isolation: the
forward 73728 x 25 x 20 and the weight gradient 25 x 73728 x 20, timed per
launch (CUDA events on the launching stream) - for ncu and A/B runs
(MPX_THIN=0 selects the tiled SIMT kernel)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2402_02320_b200 import _lib
from paper_2402_02320_b200.protocols import batch_matmul
from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
from paper_2402_02320_b200.session import SimSession

n = int(os.environ.get("N", 3))
rng = np.random.default_rng(1)
cols = rng.integers(0, 1 << 64, (73728, 25), dtype=np.uint64)
W = rng.integers(0, 1 << 64, (25, 20), dtype=np.uint64)
dz = rng.integers(0, 1 << 64, (73728, 20), dtype=np.uint64)


def run(s):
    x = s.share_ring(cols, 64, 0, [1, 1])
    w = s.share_ring(W, 64, 0, [1, 2])
    g = s.share_ring(dz, 64, 0, [1, 3])
    xt = type(x).strided(x.values.transpose(-1, -2), 64, 0, x.parties)
    z1 = batch_matmul(s, [(x, w)])[0]
    z2 = batch_matmul(s, [(xt, g)])[0]
    return z1, z2


c = DemandCounter(tuple(range(n)), n)
run(SimSession(n, c))
for rep in range(3):
    s = SimSession(n, device_store(7 + rep, n, c.demands, needs_bits=c.needs_bits))
    torch.cuda.synchronize()
    _lib.profile_begin()
    z1, z2 = run(s)
    torch.cuda.synchronize()
    prof = _lib.profile_end()
    print(" ".join(f"{nm}:{1e3 * a.elapsed_time(b):.1f}us" for nm, _, a, b in prof if "gemm" in nm or "mask" in nm))
