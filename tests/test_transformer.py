"""Secure Transformer inference (configs[3] stand-in).

CPU: the B200 forward's dry run requests the oracle restatement's material
and ledger. GPU: a small encoder (2 layers, d 32, 4 heads, FFN 64, seq 16) is
bit-exact against the oracle on every party's output shares and close to its
float64 twin; the CUDA-graphed forward equals the eager forward.
"""

import numpy as np
import pytest
import torch

import oracle as O
from oracle import transformer_sim as OT

CFG = dict(layers=2, d=32, heads=4, ffn=64, frac=14)
S = 16


def _x(seed=4):
    return np.random.default_rng(seed).normal(0, 1, (S, CFG["d"]))


def test_transformer_dry_run_matches_oracle():
    from paper_2402_02320_b200.preprocessing import DemandCounter
    from paper_2402_02320_b200.session import SimSession, demands_by_name
    from paper_2402_02320_b200.transformer import Transformer
    n = 2
    c = DemandCounter((0, 1), n)
    s = SimSession(n, c)
    m = Transformer(s, **CFG)
    m.forward(s, s.share_fixed(_x(), 64, 14, [9, 9]))
    od = O.Sim(n, O.Demand(n))
    om = OT.Transformer(od, **CFG)
    om.forward(od, OT.share_fixed(od, _x(), 64, 14, [9, 9]))
    assert demands_by_name(c) == dict(sorted(od.store.demands.items()))
    assert {k: v.as_dict() for k, v in s.metrics.ledger.items()} == \
        {k: v.as_dict() for k, v in od.ledger.by_scope.items()}
    assert Transformer(SimSession(n, DemandCounter((0, 1), n)), layers=6).n_params == 18_874_368


@pytest.mark.gpu
def test_transformer_bit_exact_and_accurate():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200.preprocessing import DemandCounter, device_store
    from paper_2402_02320_b200.session import SimSession
    from paper_2402_02320_b200.transformer import GraphedInference, Transformer
    n = 2
    c = DemandCounter((0, 1), n)
    sd = SimSession(n, c)
    Transformer(sd, **CFG).forward(sd, sd.share_fixed(_x(), 64, 14, [9, 9]))
    s = SimSession(n, device_store(11, n, c.demands, needs_bits=c.needs_bits))
    m = Transformer(s, **CFG)
    xs = s.share_fixed(_x(), 64, 14, [9, 9])
    y = m.forward(s, xs)
    torch.cuda.synchronize()

    def ofn(so):
        om = OT.Transformer(so, **CFG)
        return om.forward(so, OT.share_fixed(so, _x(), 64, 14, [9, 9]))
    want, _ = O.simulate(ofn, n, 11)
    assert np.array_equal(y.values.cpu().numpy().view(np.uint64), want.values)
    got = s.open_fixed(y)
    xq = np.floor(_x() * (1 << 14)) / (1 << 14)
    assert np.abs(got - m.plaintext(xq)).max() < 2e-2

    # graphed == eager with the same re-dealt material
    g = GraphedInference(s, m, xs, c.demands, c.needs_bits, seed0=11)
    yg = g.run(11)
    torch.cuda.synchronize()
    assert torch.equal(yg.values, y.values)
