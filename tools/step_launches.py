"""Per-launch table of one eager training step (CUDA events around every
libmpx call on the launching stream), with the algorithmic bytes / int8 ops
bench.py attributes to each launch.

    python tools/step_launches.py [--arch lenet|alexnet|vgg16m] [--parties 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2402_02320_b200 import _lib, train  # noqa: E402
from paper_2402_02320_b200.preprocessing import DemandCounter, device_store  # noqa: E402
from paper_2402_02320_b200.session import SimSession  # noqa: E402


def _table(prof_runs):
    rows = None
    for prof in prof_runs:
        cur = []
        for name, args, e0, e1 in prof:
            us = 1e3 * e0.elapsed_time(e1)
            b = bench.alg_bytes(name, args)
            ops = None
            if name == "mpx_gemm_limbs":
                ops = 2 * 36 * args[3] * args[4] * args[5] * args[8]
            elif name == "mpx_gemm_limbs_split":
                ops = 2 * 36 * args[5] * args[6] * args[7] * 2 * args[10]
            short = [v for v in args if isinstance(v, int) and abs(v) < 1 << 40][:12]
            cur.append([name, short, us, b, ops])
        if rows is None:
            rows = cur
        else:
            for r, c_ in zip(rows, cur):
                r[2] = min(r[2], c_[2])
    return rows


def _print(rows, full=True):
    tot = sum(r[2] for r in rows)
    if full:
        for name, short, us, b, ops in rows:
            extra = ""
            if b:
                extra = f"{b / 1e6:9.1f} MB {b / us / 1e3:7.0f} GB/s"
            if ops:
                extra = f"{ops / 1e9:9.1f} Gop {ops / us / 1e6:7.0f} TOPS"
            print(f"{us:8.1f} us {100 * us / tot:5.1f}%  {name:28s} {extra:30s} {short}")
    print(f"total {tot:.1f} us, {len(rows)} launches")
    agg = {}
    for name, _, us, _, _ in rows:
        agg[name] = agg.get(name, 0) + us
    print(json.dumps({k: round(v, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])}))


def transformer(a, dev):
    from paper_2402_02320_b200.transformer import Transformer
    n, S = a.parties, 128
    x = np.random.default_rng(3).normal(0, 1, (S, 512))
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c, device=dev)
    Transformer(sd).forward(sd, sd.share_fixed(x, 64, 14, [5, 5]))
    s = SimSession(n, None, device=dev)
    m = Transformer(s)
    xs = s.share_fixed(x, 64, 14, [5, 5])
    runs = []
    for rep in range(a.reps):
        s.store = device_store(60 + rep, n, c.demands, device=dev, needs_bits=c.needs_bits)
        torch.cuda.synchronize()
        _lib.profile_begin()
        m.forward(s, xs)
        torch.cuda.synchronize()
        runs.append(_lib.profile_end())
    rows = _table(runs)
    _print(rows, full=not a.summary)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="lenet")
    ap.add_argument("--parties", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--summary", action="store_true")
    a = ap.parse_args()
    n = a.parties
    dev = torch.device("cuda", 0)
    if a.arch == "transformer":
        return transformer(a, dev)
    if a.arch == "lenet":
        x, y = bench.lenet_data(bench.BATCH)
    else:
        rng = np.random.default_rng(6)
        x, y = rng.uniform(0, 1, (bench.BATCH, 3, 32, 32)), np.eye(10)[rng.integers(0, 10, bench.BATCH)]
    build = getattr(train, a.arch)
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c, device=dev)
    md = build(sd)
    p = md.layers[0].p
    md.train_step(sd, sd.share_fixed(x, 64, p, [2, 1]), sd.share_fixed(y, 64, p, [2, 2]), bench.LR_SHIFT)
    s = SimSession(n, None, device=dev)
    m = build(s)
    xs, ys = s.share_fixed(x, 64, p, [2, 1]), s.share_fixed(y, 64, p, [2, 2])
    runs = []
    for rep in range(a.reps):
        s.store = device_store(50 + rep, n, c.demands, device=dev, needs_bits=c.needs_bits)
        torch.cuda.synchronize()
        _lib.profile_begin()
        m.train_step(s, xs, ys, bench.LR_SHIFT)
        torch.cuda.synchronize()
        runs.append(_lib.profile_end())
        del s.store
    _print(_table(runs), full=not a.summary)


if __name__ == "__main__":
    main()
