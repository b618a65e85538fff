"""Golden digests of the oracle at the EXACT bench configurations (this container).

    python tests/golden/make_bench_fixtures.py [lenet_n3_b128] [transformer_n2_s128] ...

The bench workloads are too large to store every party's output shares
(LeNet's weights alone are 10 MB per step), so this script runs the pinned
oracle (``oracle/``, itself bit-exact against reference-generated fixtures)
on the bench's own inputs, keys and dealer seed 11 and stores, per output
tensor, the SHA-256 of every party's uint64 share words (party-major,
little-endian) plus a few plain words for diagnostics. The ``-m gpu`` tests in
``tests/test_bench_configs.py`` run the same configuration through the C-ABI
and compare digests: bit-exact or fail.

Cases (BASELINE.json configs):
* ``lenet_n3_b128``: configs[1] - one LeNet SGD step, 3 parties, batch 128
  (bench.py's ``lenet_data(128)`` and share keys), every party's logits and
  every layer's W / b after the update.
* ``transformer_n2_s128``: configs[3] - the full 18,874,368-weight encoder
  (6 layers, d 512, 8 heads, FFN 2048, p = 14), seq 128, 2 parties, output
  shares of the forward pass.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

OUT = os.path.join(HERE, "bench_configs.json")


def digest(u64: np.ndarray) -> dict:
    a = np.ascontiguousarray(np.asarray(u64).view(np.uint64))
    return {"sha256": hashlib.sha256(a.astype("<u8").tobytes()).hexdigest(), "shape": list(a.shape),
            "head": [int(v) for v in a.reshape(-1)[:4]]}


def lenet_n3_b128():
    import oracle as O
    from oracle import train_sim as OT
    import bench
    n, B = 3, bench.BATCH
    x, y = bench.lenet_data(B)

    def fn(s):
        m = OT.lenet(s)
        xs = OT.share_fixed(s, x, bench.WIDTH, bench.FRAC, bench.label_key("share:x"))
        ys = OT.share_fixed(s, y, bench.WIDTH, bench.FRAC, bench.label_key("share:y"))
        return m, m.train_step(s, xs, ys, bench.LR_SHIFT)

    (m, logits), _ = O.simulate(fn, n, 11)
    out = {"logits": digest(logits.values)}
    for i, layer in enumerate(m.layers):
        for attr in ("W", "b"):
            if hasattr(layer, attr):
                out[f"{i}.{attr}"] = digest(getattr(layer, attr).values)
    return {"n": n, "batch": B, "seed": 11, "outputs": out}


def transformer_n2_s128():
    import oracle as O
    from oracle import transformer_sim as OT
    n, S = 2, 128
    x = np.random.default_rng(3).normal(0, 1, (S, 512))

    def fn(s):
        m = OT.Transformer(s)
        return m.forward(s, OT.share_fixed(s, x, 64, 14, [5, 5]))

    y, _ = O.simulate(fn, n, 11)
    return {"n": n, "seq": S, "seed": 11, "outputs": {"y": digest(y.values)}}


CASES = {"lenet_n3_b128": lenet_n3_b128, "transformer_n2_s128": transformer_n2_s128}


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for nm in names or list(CASES):
        t0 = time.time()
        data[nm] = CASES[nm]()
        data[nm]["oracle_seconds"] = round(time.time() - t0, 1)
        print(nm, data[nm]["oracle_seconds"], "s", flush=True)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
