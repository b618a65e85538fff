"""The reference arm of bench.py (``baseline/reference_arm.py``) runs the
UNMODIFIED reference package from ``baseline/_ref``; its LeNet step (the
oracle's training composition over the reference's per-party primitives) is
bit-exact with the oracle - and so with the GPU engine - on every party's
logits and weights. Skipped when the reference install is absent."""

import numpy as np
import pytest

import oracle as O
from oracle import train_sim as OT

ra = pytest.importorskip("baseline.reference_arm")
if ra.available() is not None:
    pytest.skip(ra.available(), allow_module_level=True)


@pytest.mark.slow
def test_reference_lenet_step_matches_oracle():
    import bench
    n, B = 3, 2
    x, y = bench.lenet_data(B)
    keys = (bench.label_key("share:x"), bench.label_key("share:y"))
    outs, secs = ra.lenet_step(x, y, n, keys)
    assert secs > 0

    def fn(s):
        m = OT.lenet(s)
        xs = OT.share_fixed(s, x, 64, 23, keys[0])
        ys = OT.share_fixed(s, y, 64, 23, keys[1])
        return m, m.train_step(s, xs, ys, bench.LR_SHIFT)

    (om, ol), _ = O.simulate(fn, n, 11)
    assert np.array_equal(np.stack([o[1].values for o in outs]), ol.values)
    for li, layer in enumerate(om.layers):
        if hasattr(layer, "W"):
            got = np.stack([o[0].layers[li].W.values for o in outs])
            assert np.array_equal(got, layer.W.values), li


def test_reference_reciprocal_matches_oracle():
    import bench
    enc = bench.encode_np(bench.workload_inputs(300))
    key = bench.label_key("share:x")
    outs, _ = ra.reciprocal_sample(enc, 2, key)

    def fn(s):
        return O.reciprocal(s, O.AShare(O.deal_inputs_arith(enc, 2, 64, key), 64, 23))

    want, _ = O.simulate(fn, 2, 11)
    assert np.array_equal(np.stack([o.values for o in outs]), want.values)


@pytest.mark.slow
def test_reference_alexnet_step_matches_oracle():
    """configs[2] composition (bias, strided / padded convs, 3x3/2 pool) on the reference."""
    n, B = 2, 1
    rng = np.random.default_rng(6)
    x, y = rng.uniform(0, 1, (B, 3, 32, 32)), np.eye(10)[rng.integers(0, 10, B)]
    keys = ([2, 1], [2, 2])
    outs, _ = ra.train_step("alexnet", x, y, n, keys)

    def fn(s):
        m = OT.alexnet(s)
        return m, m.train_step(s, OT.share_fixed(s, x, 64, 23, keys[0]), OT.share_fixed(s, y, 64, 23, keys[1]), 5)

    (om, ol), _ = O.simulate(fn, n, 11)
    assert np.array_equal(np.stack([o[1].values for o in outs]), ol.values)
    for li, layer in enumerate(om.layers):
        for nm in ("W", "b"):
            if getattr(layer, nm, None) is not None:
                assert np.array_equal(np.stack([getattr(o[0].layers[li], nm).values for o in outs]),
                                      getattr(layer, nm).values), (li, nm)


@pytest.mark.slow
def test_reference_transformer_matches_oracle():
    from oracle import transformer_sim as OTS
    cfg = dict(layers=1, d=32, heads=4, ffn=64, frac=14)
    x = np.random.default_rng(4).normal(0, 1, (16, 32))
    outs, _ = ra.transformer_forward(x, 2, key=(9, 9), **cfg)

    def fn(s):
        return OTS.Transformer(s, **cfg).forward(s, OTS.share_fixed(s, x, 64, 14, [9, 9]))

    want, _ = O.simulate(fn, 2, 11)
    assert np.array_equal(np.stack([o.values for o in outs]), want.values)
