"""One online step of a secure op under an NVTX range named "online", for ncu.

    python tools/profile_step.py [--op reciprocal|exp|log|mul|matmul] [--elems N] [--parties n]

Deals material, runs one warm-up step, deals again, then runs one step inside
``torch.cuda.nvtx.range("online")`` so ``ncu --nvtx --nvtx-include online/``
captures exactly the kernels of one step.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2402_02320_b200 as G  # noqa: E402
from paper_2402_02320_b200.preprocessing import DemandCounter, device_store  # noqa: E402
from paper_2402_02320_b200.protocols import batch_matmul, mul  # noqa: E402
from paper_2402_02320_b200.session import SimSession  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="reciprocal")
    ap.add_argument("--elems", type=int, default=1 << 24)
    ap.add_argument("--parties", type=int, default=2)
    ap.add_argument("--dim", type=int, default=4096)
    args = ap.parse_args()
    n = args.parties
    rng = np.random.default_rng(1)
    if args.op == "reciprocal":
        xs = np.exp2(rng.uniform(-8, 8, args.elems)) * rng.choice([-1.0, 1.0], args.elems)
    elif args.op == "exp":
        xs = rng.uniform(-16, 16, args.elems)
    elif args.op == "log":
        xs = np.exp2(rng.uniform(-8, 8, args.elems))
    else:
        xs = rng.uniform(-4, 4, args.elems)
    enc = np.floor(xs * (1 << 23)).astype(np.int64).view(np.uint64)

    def op(s, x, y=None):
        if args.op == "reciprocal":
            return G.reciprocal(s, x)
        if args.op == "exp":
            return G.exponentiation(s, x)
        if args.op == "log":
            return G.logarithm(s, x)
        if args.op == "mul":
            return mul(s, x, y)
        if args.op == "matmul":
            return batch_matmul(s, [(x, y)])[0]
        raise SystemExit(f"unknown op {args.op}")

    def inputs(s):
        if args.op == "matmul":
            d = args.dim
            a = rng.integers(0, 1 << 64, (d, d), dtype=np.uint64)
            return s.share_ring(a, 64, 0, [1, 2]), s.share_ring(a, 64, 0, [3, 4])
        x = s.share_ring(enc, 64, 23, [1000, 2])
        return x, x

    counter = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, counter)
    op(sd, *inputs(sd))
    s0 = SimSession(n, None)
    x, y = inputs(s0)
    for step in range(2):
        store = device_store(100 + step, n, counter.demands, needs_bits=counter.needs_bits)
        s = SimSession(n, store)
        torch.cuda.synchronize()
        if step == 1:
            with torch.cuda.nvtx.range("online"):
                op(s, x, y)
        else:
            op(s, x, y)
        torch.cuda.synchronize()
        del store, s
    print("ok")


if __name__ == "__main__":
    main()
