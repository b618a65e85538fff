"""GPU parity: the B200 path (through the libmpx C ABI) against the reference
golden fixtures and the CPU oracle — bit-exact shares for every party.

Every case: dry run -> on-device Philox dealer -> live sim-mode run; each
party's output shares must equal the reference's bit for bit (golden
fixtures, which the oracle is pinned to) and, at larger sizes, the oracle's.
"""

import json
import os

import numpy as np
import pytest
import torch

from cases import CASES

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def engine():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from gpu_engine import GpuEngine
    return GpuEngine()


@pytest.fixture(scope="module")
def oracle_engine():
    from engines import OracleEngine
    return OracleEngine()


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case_bit_exact(engine, name):
    fn, n = CASES[name]
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    info = json.loads(bytes(z["info"]).decode())
    got, ginfo, _ = engine.run(fn, n)
    assert ginfo["demands"] == info["demands"]
    assert ginfo["total"] == info["total"]
    for k, v in got.items():
        want = z[f"out__{k}"]
        assert v.shape == want.shape, (k, v.shape, want.shape)
        assert np.array_equal(v, want), (k, np.argwhere(v != want)[:5])


def test_dealer_matches_reference_generate_material(engine):
    from paper_2402_02320_b200.preprocessing import Dealer, MaterialKey
    z = np.load(os.path.join(GOLDEN, "dealer.npz"))
    groups = {}
    for k in z.files:
        name, count, arr = k.split("__")
        groups.setdefault((name, int(count)), {})[arr] = z[k]
    d = Dealer(11, 3, 0, 3, "cuda")
    for (name, count), arrays in groups.items():
        key = MaterialKey.from_name(name)
        got = d.generate(key, count, need_bits=True)
        for arr, want in arrays.items():
            g = got[arr].cpu().numpy()
            if want.dtype == np.uint8:   # packed bit stream -> one byte per bit
                flat = np.unpackbits(g.view(np.uint8), axis=-1, bitorder="little")
                g = flat[:, :want[0].size].reshape(want.shape)
            else:
                g = g.view(np.uint64).reshape(want.shape)
            assert np.array_equal(g, want), (name, arr)


def _compare(engine, oracle_engine, fn, n, seed=11):
    got, ginfo, _ = engine.run(fn, n, seed)
    want, winfo = oracle_engine.run(fn, n, seed)
    assert ginfo["demands"] == winfo["demands"]
    assert ginfo["total"] == winfo["total"]
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    return got


def big_mul(M, s):
    rng = np.random.default_rng(5)
    xs = rng.integers(0, 1 << 64, 1 << 16, dtype=np.uint64)
    ys = rng.integers(0, 1 << 64, 1 << 16, dtype=np.uint64)
    return {"z": M.mul(s, M.deal_arith(s, xs, 64, tag=0), M.deal_arith(s, ys, 64, tag=1))}


def big_matmul(M, s):
    rng = np.random.default_rng(6)
    a = rng.integers(0, 1 << 64, (96, 160), dtype=np.uint64)
    b = rng.integers(0, 1 << 64, (160, 72), dtype=np.uint64)
    return {"z": M.batch_matmul(s, [(M.deal_arith(s, a, 64, tag=0), M.deal_arith(s, b, 64, tag=1))])[0]}


def tc_matmul(M, s):
    rng = np.random.default_rng(16)
    a = rng.integers(0, 1 << 64, (256, 320), dtype=np.uint64)
    b = rng.integers(0, 1 << 64, (320, 192), dtype=np.uint64)
    c = rng.integers(0, 1 << 64, (130, 256), dtype=np.uint64)
    d = rng.integers(0, 1 << 64, (256, 96), dtype=np.uint64)
    return {f"z{i}": z for i, z in enumerate(M.batch_matmul(s, [
        (M.deal_arith(s, a, 64, tag=0), M.deal_arith(s, b, 64, tag=1)),
        (M.deal_arith(s, c, 64, tag=2), M.deal_arith(s, d, 64, tag=3))]))}


def big_decompose(M, s):
    rng = np.random.default_rng(7)
    xs = rng.integers(0, 1 << 64, 20000, dtype=np.uint64)
    return {"bits": M.decompose(s, M.deal_arith(s, xs, 64, tag=0))}


def big_reciprocal(M, s):
    rng = np.random.default_rng(8)
    xs = np.exp2(rng.uniform(-8, 8, 4096)) * rng.choice([-1.0, 1.0], 4096)
    return {"y": M.reciprocal(s, M.deal_fixed(s, xs, 64, 23, tag=0))}


def big_exp(M, s):
    rng = np.random.default_rng(9)
    return {"y": M.exponentiation(s, M.deal_fixed(s, rng.uniform(-16, 16, 4096), 64, 23, tag=0))}


def big_log(M, s):
    rng = np.random.default_rng(10)
    return {"y": M.logarithm(s, M.deal_fixed(s, np.exp2(rng.uniform(-8, 8, 4096)), 64, 23, tag=0))}


def big_softmax(M, s):
    rng = np.random.default_rng(11)
    return {"y": M.softmax(s, M.deal_fixed(s, rng.normal(0, 4, (16, 128)), 64, 14, tag=0))}


def big_attention(M, s):
    rng = np.random.default_rng(12)
    heads = []
    for h in range(2):
        q, k, v = rng.normal(0, 1, (32, 16)), rng.normal(0, 1, (32, 16)), rng.normal(0, 0.5, (32, 16))
        heads.append((M.deal_fixed(s, q, 64, 14, tag=3 * h),
                      M.deal_fixed(s, k * 1.4426950408889634 / 4.0, 64, 14, tag=3 * h + 1),
                      M.deal_fixed(s, v, 64, 14, tag=3 * h + 2)))
    return {"o": M.attention_block(s, heads, optimized=True)}


@pytest.mark.parametrize("fn,n", [(big_mul, 3), (big_matmul, 2), (tc_matmul, 2), (tc_matmul, 3),
                                  (big_decompose, 4),
                                  (big_reciprocal, 2), (big_exp, 3), (big_log, 2),
                                  (big_softmax, 2), (big_attention, 2)],
                         ids=["mul65536_n3", "matmul96x160x72", "tc_matmul_n2", "tc_matmul_n3", "decompose20000_n4", "reciprocal4096",
                              "exp4096_n3", "log4096", "softmax16x128", "attention2h32"])
def test_larger_sizes_vs_oracle(engine, oracle_engine, fn, n):
    _compare(engine, oracle_engine, fn, n)


def test_reciprocal_accuracy_budget(engine):
    """Criterion 3 budget (tests/test_acceptance.py:135): rel err <= 1e-4."""
    from paper_2402_02320_b200.ring import decode
    xs = np.concatenate([np.logspace(-8, 8, 200, base=2), -np.logspace(-8, 8, 200, base=2)])

    def fn(M, s):
        return {"y": M.reciprocal(s, M.deal_fixed(s, xs, 64, 23, tag=0))}
    got, _, sess = engine.run(fn, 2)
    y = got["y"]
    opened = (y[0] + y[1]).view(np.int64) / float(1 << 23)
    xq = np.floor(xs * (1 << 23)) / (1 << 23)
    rel = np.abs(opened - 1 / xq) * np.abs(xq)
    assert rel.max() <= 1e-4, rel.max()
