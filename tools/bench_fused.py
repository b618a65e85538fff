"""Time the sim-mode fused kernels alone (Reciprocal/Exp/Log/ReLU/max_vec;
default 2 parties, 2^24 elements).

    python tools/bench_fused.py [--kinds relu,max_vec] [--parties 3] [--elems N]
"""
import argparse, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02320_b200 as G  # noqa: E402
from paper_2402_02320_b200.protocols import max_vec as MV  # noqa: E402
from paper_2402_02320_b200.preprocessing import DemandCounter, device_store  # noqa: E402
from paper_2402_02320_b200.session import SimSession  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--parties", type=int, default=2)
    ap.add_argument("--kinds", default="reciprocal,exp,log")
    a = ap.parse_args()
    n = a.parties
    rng = np.random.default_rng(3)
    out = {}
    for kind, fn, xs in (("reciprocal", G.reciprocal, np.exp2(rng.uniform(-8, 8, a.elems))),
                         ("exp", G.exponentiation, rng.uniform(-16, 16, a.elems)),
                         ("log", G.logarithm, np.exp2(rng.uniform(-8, 8, a.elems))),
                         ("relu", G.relu, rng.normal(0, 4, a.elems)),
                         ("max_vec", lambda s, x: MV(s, x.reshape((a.elems // 64, 64))),
                          rng.normal(0, 4, a.elems))):
        if kind not in a.kinds.split(","):
            continue
        enc = np.floor(xs * (1 << 23)).astype(np.int64).view(np.uint64)
        c = DemandCounter(tuple(range(n)), n)
        sd = SimSession(n, c)
        fn(sd, sd.share_ring(enc, 64, 23, [1, 2]))
        x = SimSession(n, None).share_ring(enc, 64, 23, [1, 2])
        ts = []
        for r in range(a.reps + 1):
            st = device_store(7 + r, n, c.demands, needs_bits=c.needs_bits)
            s = SimSession(n, st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(s, x)
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
            del st, s
        out[kind] = round(min(ts), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
