"""GPU: sim-mode whole-op fused kernels (one kernel per Reciprocal / Exp /
Log) are bit-exact against the per-round path and the CPU oracle, consume the
same material (store usage) and record the same ledger."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engines():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from engines import OracleEngine
    from gpu_engine import GpuEngine
    return GpuEngine(), OracleEngine()


def _recip(M, s):
    rng = np.random.default_rng(21)
    xs = np.exp2(rng.uniform(-8, 8, 6000)) * rng.choice([-1.0, 1.0], 6000)
    return {"y": M.reciprocal(s, M.deal_fixed(s, xs, 64, 23, tag=0))}


def _exp(M, s):
    rng = np.random.default_rng(22)
    return {"y": M.exponentiation(s, M.deal_fixed(s, rng.uniform(-16, 16, 6000), 64, 23, tag=0))}


def _exp14(M, s):
    rng = np.random.default_rng(23)
    return {"y": M.exponentiation(s, M.deal_fixed(s, rng.uniform(-10, 5, 3000), 64, 14, tag=0))}


def _log(M, s):
    rng = np.random.default_rng(24)
    return {"y": M.logarithm(s, M.deal_fixed(s, np.exp2(rng.uniform(-8, 8, 6000)), 64, 23, tag=0))}


def _chain(M, s):
    """ops back to back share the material keys: cursors must line up"""
    rng = np.random.default_rng(25)
    x = M.deal_fixed(s, rng.uniform(0.5, 4.0, 2000), 64, 23, tag=0)
    y = M.exponentiation(s, M.logarithm(s, x))
    return {"y": y, "r": M.reciprocal(s, y)}


@pytest.mark.parametrize("fn", [_recip, _exp, _exp14, _log, _chain], ids=["recip", "exp", "exp_p14", "log", "chain"])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_fused_equals_per_round_and_oracle(engines, fn, n):
    g, o = engines
    fused, finfo, fs = g.run(fn, n, fuse=True)
    rounds, rinfo, rs = g.run(fn, n, fuse=False)
    want, winfo = o.run(fn, n)
    assert finfo["ledger"] == rinfo["ledger"] == winfo["ledger"]
    assert fs.store.usage() == rs.store.usage()
    for k in want:
        assert np.array_equal(fused[k], want[k]), k
        assert np.array_equal(rounds[k], want[k]), k


def _relu(M, s):
    rng = np.random.default_rng(26)
    return {"y": M.relu(s, M.deal_fixed(s, rng.normal(0, 4, 5000), 64, 23, tag=0))}


def _relu32(M, s):
    rng = np.random.default_rng(27)
    return {"y": M.relu(s, M.deal_fixed(s, rng.normal(0, 4, (40, 33)), 32, 14, tag=0))}


def _max_odd(M, s):
    rng = np.random.default_rng(28)
    return {"m": M.max_vec(s, M.deal_fixed(s, rng.normal(0, 5, (37, 23)), 64, 23, tag=0))}


def _maxcut_softmax(M, s):
    rng = np.random.default_rng(29)
    x = M.deal_fixed(s, rng.normal(0, 5, (9, 64)), 64, 23, tag=0)
    return {"mc": M.maxcut(s, x), "sm": M.softmax(s, x)}


def _attexp(M, s):
    rng = np.random.default_rng(30)
    x = M.deal_fixed(s, -np.abs(rng.normal(0, 6, 3000)) - 2 ** -23, 32, 23, tag=0)
    return {"y": M.attention_exp(s, x)}


def _attexp14(M, s):
    rng = np.random.default_rng(31)
    x = M.deal_fixed(s, -np.abs(rng.normal(0, 4, (16, 40))), 32, 14, tag=0)
    return {"y": M.attention_exp(s, x)}


def _attention(M, s):
    rng = np.random.default_rng(32)
    heads = []
    for h in range(2):
        q, k, v = (M.deal_fixed(s, rng.normal(0, 1, (24, 16)), 64, 14, tag=3 * h + i) for i in range(3))
        heads.append((q, k, v))
    return {"a": M.attention_block(s, heads, optimized=True)}


@pytest.mark.parametrize("fn", [_relu, _relu32, _max_odd, _maxcut_softmax, _attexp, _attexp14, _attention],
                         ids=["relu", "relu_w32", "max_odd", "maxcut_softmax", "attexp", "attexp_p14",
                              "attention"])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_fused_cmp_equals_per_round_and_oracle(engines, fn, n):
    g, o = engines
    fused, finfo, fs = g.run(fn, n, fuse=True)
    rounds, rinfo, rs = g.run(fn, n, fuse=False)
    want, winfo = o.run(fn, n)
    assert finfo["ledger"] == rinfo["ledger"] == winfo["ledger"]
    assert fs.store.usage() == rs.store.usage()
    for k in want:
        assert np.array_equal(fused[k], want[k]), k
        assert np.array_equal(rounds[k], want[k]), k

