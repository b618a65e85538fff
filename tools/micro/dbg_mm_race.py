"""Repeat the acceptance batch_matmul (25 x 20x20 @ 20x20, party threads) and report mismatches."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from mpfix_helpers import deal_arith, run_mpc
from paper_2402_02320_b200.mpfix.protocols import batch_matmul


def fn(session):
    rng = np.random.default_rng(1)
    a_mats = rng.integers(0, 1 << 64, (25, 20, 20), dtype=np.uint64)
    b_mats = rng.integers(0, 1 << 64, (25, 20, 20), dtype=np.uint64)
    pairs = [(deal_arith(session, a_mats[i], 64, tag=100 + 2 * i), deal_arith(session, b_mats[i], 64, tag=101 + 2 * i))
             for i in range(25)]
    got = np.stack([session.open_arith(o) for o in batch_matmul(session, pairs)])
    return got, np.matmul(a_mats, b_mats)


for n in (2, 3, 5):
    fails = 0
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
        res = run_mpc(fn, n)
        for p, (g, w) in enumerate(res):
            if not np.array_equal(g, w):
                fails += 1
                bad = np.argwhere(g != w)
                print(f"n={n} it={it} party={p} bad={len(bad)} pairs={sorted(set(bad[:, 0].tolist()))[:10]}")
    print(f"n={n}: {fails} failing party results")
