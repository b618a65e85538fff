"""Bit-exact parity AT THE BENCH CONFIGURATIONS (BASELINE.json configs[1], [3], [4]).

The smaller parity tests route differently from the benchmarked shapes (SIMT
vs tcgen05 GEMMs, split-K, staged epilogues, fused vs per-round paths), so
these run the exact workloads ``bench.py`` times:

* configs[1]: one LeNet SGD step, 3 parties, batch 128 (bench inputs and
  keys, dealer seed 11) - eager AND replayed from the CUDA graph - against
  SHA-256 digests of the oracle's shares (``tests/golden/bench_configs.json``,
  made by ``tests/golden/make_bench_fixtures.py``);
* configs[3]: the full 18,874,368-weight Transformer at seq 128, 2 parties,
  eager and graphed, against the oracle's digest;
* configs[4]: Reciprocal / Exp / Log on 2^24 elements (n = 2) and 2^22
  (n = 8): the whole-op fused kernel == the per-round path, share for share,
  and the decoded outputs meet the reference's accuracy budgets
  (tests/test_acceptance.py:131-139 of the reference: reciprocal rel <= 1e-4,
  exp scaled <= 1e-4, log abs <= 1e-3) over the benchmarked input ranges;
  the 4096^3 Beaver matmul (n = 2): opened Z == X @ Y mod 2^64, checked with
  Freivalds' test on random u64 vectors (numpy's wrapping uint64 matmul, the
  reference's ring.matmul, ring.py:60-62).
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import bench

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = json.load(open(os.path.join(HERE, "golden", "bench_configs.json")))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _digest(t: torch.Tensor) -> str:
    a = np.ascontiguousarray(t.cpu().numpy().view(np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def _check(outputs: dict, want: dict):
    for k, w in want.items():
        got = outputs[k]
        assert list(got.shape) == w["shape"], (k, got.shape)
        assert _digest(got) == w["sha256"], (k, got.reshape(-1)[:4].cpu().numpy().view(np.uint64), w["head"])


def _lenet_outputs(model, logits):
    out = {"logits": logits.values}
    for i, layer in enumerate(model.layers):
        for attr in ("W", "b"):
            if hasattr(layer, attr):
                out[f"{i}.{attr}"] = getattr(layer, attr).values
    return out


def test_lenet_n3_b128_step_matches_oracle_digests():
    from paper_2402_02320_b200 import train
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    want = FIX["lenet_n3_b128"]
    n, B = want["n"], want["batch"]
    x, y = bench.lenet_data(B)
    kx, ky = bench.label_key("share:x"), bench.label_key("share:y")
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c)
    train.lenet(sd).train_step(sd, sd.share_fixed(x, 64, 23, kx), sd.share_fixed(y, 64, 23, ky), bench.LR_SHIFT)

    # eager
    s = SimSession(n, device_store(want["seed"], n, c.demands, needs_bits=c.needs_bits))
    m = train.lenet(s)
    logits = m.train_step(s, s.share_fixed(x, 64, 23, kx), s.share_fixed(y, 64, 23, ky), bench.LR_SHIFT)
    torch.cuda.synchronize()
    _check(_lenet_outputs(m, logits), want["outputs"])

    # the bench's path: one CUDA graph replay after an in-place re-deal
    s2 = SimSession(n, None)
    m2 = train.lenet(s2)
    g = train.GraphedStep(s2, m2, s2.share_fixed(x, 64, 23, kx), s2.share_fixed(y, 64, 23, ky), bench.LR_SHIFT,
                          c.demands, c.needs_bits, seed0=1)
    lg = g.step(want["seed"])
    torch.cuda.synchronize()
    _check(_lenet_outputs(m2, lg), want["outputs"])


def test_transformer_18p9m_seq128_matches_oracle_digest():
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    from paper_2402_02320_b200.transformer import GraphedInference, Transformer
    want = FIX["transformer_n2_s128"]
    n, S = want["n"], want["seq"]
    x = np.random.default_rng(3).normal(0, 1, (S, 512))
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c)
    Transformer(sd).forward(sd, sd.share_fixed(x, 64, 14, [5, 5]))
    s = SimSession(n, device_store(want["seed"], n, c.demands, needs_bits=c.needs_bits))
    m = Transformer(s)
    assert m.n_params == 18_874_368
    xs = s.share_fixed(x, 64, 14, [5, 5])
    y = m.forward(s, xs)
    torch.cuda.synchronize()
    _check({"y": y.values}, want["outputs"])
    g = GraphedInference(s, m, xs, c.demands, c.needs_bits, seed0=12)
    yg = g.run(want["seed"])
    torch.cuda.synchronize()
    _check({"y": yg.values}, want["outputs"])


def _sweep_inputs(name, N):
    if name == "reciprocal":
        return bench.workload_inputs(N)
    rng = np.random.default_rng(7)
    return rng.uniform(-16, 16, N) if name == "exp" else np.exp2(rng.uniform(-8, 8, N))


def _budget(name, got, xq):
    if name == "reciprocal":
        return float(np.max(np.abs(got - 1 / xq) * np.abs(xq))), 1e-4     # rel_err
    if name == "exp":
        ref = np.exp(xq)
        return float(np.max(np.abs(got - ref) / np.maximum(1.0, ref))), 1e-4   # err_scaled
    return float(np.max(np.abs(got - np.log(xq)))), 1e-3                   # abs_err


@pytest.mark.parametrize("n,log2n", [(2, 24), (8, 22)], ids=["n2_2p24", "n8_2p22"])
@pytest.mark.parametrize("name", ["reciprocal", "exp", "log"])
def test_sweep_fused_equals_per_round_at_bench_size(name, n, log2n):
    import paper_2402_02320_b200 as G
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    N = 1 << log2n
    enc = bench.encode_np(_sweep_inputs(name, N))
    key = bench.label_key(f"share:{name}")
    op = {"reciprocal": G.reciprocal, "exp": G.exponentiation, "log": G.logarithm}[name]
    c = DemandCounter(tuple(range(n)), n)
    sd = SimSession(n, c)
    op(sd, sd.share_ring(enc, 64, 23, key))
    outs, usage = {}, {}
    for fuse in (True, False):
        store = device_store(11, n, c.demands, needs_bits=c.needs_bits)
        s = SimSession(n, store)
        s.fuse_ops = fuse
        y = op(s, s.share_ring(enc, 64, 23, key))
        torch.cuda.synchronize()
        outs[fuse] = y
        usage[fuse] = store.usage()
        del store, s
        torch.cuda.empty_cache()
    assert usage[True] == usage[False]
    assert torch.equal(outs[True].values, outs[False].values)
    opened = outs[True].values.sum(0)          # int64 sum wraps = opening in Z_2^64
    got = opened.to(torch.float64).cpu().numpy() / float(1 << 23)   # |values| < 2^52: exact
    xq = enc.view(np.int64) / float(1 << 23)
    err, bound = _budget(name, got, xq)
    assert err <= bound, (name, err, bound)


def test_beaver_matmul_4096_freivalds():
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.protocols import batch_matmul
    from paper_2402_02320_b200.session import SimSession
    n, D = 2, 4096
    rng = np.random.default_rng(7)
    a = rng.integers(0, 1 << 64, (D, D), dtype=np.uint64)
    b = rng.integers(0, 1 << 64, (D, D), dtype=np.uint64)
    ka, kb = bench.label_key("share:mm_a"), bench.label_key("share:mm_b")
    c = DemandCounter((0, 1), n)
    sd = SimSession(n, c)
    batch_matmul(sd, [(sd.share_ring(a, 64, 0, ka), sd.share_ring(b, 64, 0, kb))])
    s = SimSession(n, device_store(11, n, c.demands, needs_bits=c.needs_bits))
    z = batch_matmul(s, [(s.share_ring(a, 64, 0, ka), s.share_ring(b, 64, 0, kb))])[0]
    Z = s.open_arith(z).cpu().numpy().view(np.uint64)
    r = np.random.default_rng(99).integers(0, 1 << 64, (D, 3), dtype=np.uint64)
    assert np.array_equal(np.matmul(Z, r), np.matmul(a, np.matmul(b, r)))
    # a flipped word must be caught
    Z[123, 456] ^= np.uint64(1 << 40)
    assert not np.array_equal(np.matmul(Z, r), np.matmul(a, np.matmul(b, r)))
