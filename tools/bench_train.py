"""Time secure training steps (sim mode, all parties on one GPU).

    python tools/bench_train.py [--model lenet|mlp] [--parties 3] [--batch 128] [--steps 3]
"""
import argparse, json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_02320_b200 import _lib, train  # noqa: E402
from paper_2402_02320_b200.preprocessing import DemandCounter, device_store  # noqa: E402
from paper_2402_02320_b200.session import SimSession  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="lenet")
    ap.add_argument("--parties", type=int, default=3)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--graph", action="store_true")
    a = ap.parse_args()
    n, B = a.parties, a.batch
    shape = {"lenet": (1, 28, 28), "mlp": (784,), "alexnet": (3, 32, 32), "vgg16m": (3, 32, 32)}[a.model]
    build = {"lenet": train.lenet, "mlp": train.simple_mlp, "alexnet": train.alexnet, "vgg16m": train.vgg16m}[a.model]
    rng = np.random.default_rng(0)
    x = rng.uniform(0, 1, (B,) + shape)
    y = np.eye(10)[rng.integers(0, 10, B)]
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c)
    m = build(sd)
    t0 = time.perf_counter()
    p = m.layers[0].p
    m.train_step(sd, sd.share_fixed(x, 64, p, [1, 2]), sd.share_fixed(y, 64, p, [3, 4]), 5)
    dry_s = time.perf_counter() - t0
    s = SimSession(n, None)
    model = build(s)
    xs, ys = s.share_fixed(x, 64, p, [1, 2]), s.share_fixed(y, 64, p, [3, 4])
    times, deal, host = [], [], []
    if a.graph:
        g = train.GraphedStep(s, model, xs, ys, 5, c.demands, c.needs_bits, seed0=50)
        for t in range(a.steps + 1):
            torch.cuda.synchronize()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record()
            g.dealer.redeal(60 + t)            # the dealer's CUDA graph
            d1.record()
            torch.cuda.synchronize()
            deal.append(d0.elapsed_time(d1) / 1e3)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0 = time.perf_counter()
            e0.record()
            g.graph.replay()
            e1.record()
            h1 = time.perf_counter()
            torch.cuda.synchronize()
            if t:
                times.append(e0.elapsed_time(e1))
                host.append((h1 - h0) * 1e3)
        a.steps = -1
    for t in range(a.steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.store = device_store(50 + t, n, c.demands, needs_bits=c.needs_bits)
        torch.cuda.synchronize()
        deal.append(time.perf_counter() - t0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if a.profile and t == a.steps:
            _lib.profile_begin()
        h0 = time.perf_counter()
        e0.record()
        model.train_step(s, xs, ys, 5)
        e1.record()
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        if t:
            times.append(e0.elapsed_time(e1))
            host.append((h1 - h0) * 1e3)
    mat = sum(t.numel() * t.element_size() for d in s.store._arrays.values() for t in d.values())
    out = {"material_GB": mat / 1e9, "params": model.n_params, "graph": a.graph, "model": a.model, "parties": n, "batch": B, "ms_per_step": float(np.mean(times)),
           "steps_per_s": 1e3 / float(np.mean(times)), "host_issue_ms": float(np.mean(host)),
           "dealer_ms": 1e3 * float(np.mean(deal[1:])), "dry_run_s": dry_s,
           "rounds_per_step": s.metrics.total.rounds // max(1, a.steps + 1),
           "launches_per_step": None}
    if a.profile:
        prof = _lib.profile_end()
        agg = {}
        for nm, _a, p0, p1 in prof:
            d = agg.setdefault(nm, [0.0, 0])
            d[0] += p0.elapsed_time(p1)
            d[1] += 1
        out["launches_per_step"] = sum(v[1] for v in agg.values())
        out["kernels"] = {k: [round(v[0], 3), v[1]] for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
