"""The reference-compatible facade (``paper_2402_02320_b200.mpfix``), SURVEY §8b.

CPU: the facade exports the reference's public names with the reference's
parameter names (``__init__.py:5-45``, ``protocols/__init__.py:1-30``,
SURVEY §8b signature table) and ``install()`` makes ``import mpfix`` resolve
to it. GPU: every golden case (fixtures produced by running the reference)
driven through the facade exactly as the reference's own tests drive
``mpfix`` - a party thread per party, numpy handles - is bit-exact on every
party's shares, with the reference's material demand and ledger.
"""

import inspect
import json
import os
import sys

import numpy as np
import pytest

from cases import CASES

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SIGNATURES = {
    "protocols": {"mul": ["session", "x", "y"], "matmul": ["session", "x", "y"],
                  "batch_matmul": ["session", "pairs"], "and_gate": ["session", "x", "y"],
                  "binary_add": ["session", "x", "y"], "public_add_bits": ["session", "pub_bits", "x"],
                  "bit2a": ["session", "b", "width"], "compose": ["session", "bits", "width", "frac"],
                  "decompose": ["session", "x"], "gt": ["session", "x", "y"],
                  "const_share": ["session", "value", "width", "frac", "shape"],
                  "add_const": ["session", "x", "value"], "truncate": ["session", "x", "f", "out_frac"],
                  "unsigned_truncate": ["session", "x", "f", "out_frac"],
                  "scale_fixed": ["session", "x", "const", "const_frac"],
                  "evaluate_poly": ["session", "x", "coeffs", "frac"],
                  "evaluate_square_completed": ["session", "x", "lead_shift", "t3", "t2", "lin_coeff",
                                                "const_coeff", "frac"],
                  "lmo": ["session", "bits"], "max_vec": ["session", "x"]},
    "nonlinear": {"reciprocal": ["session", "x", "params"], "exponentiation": ["session", "x", "params"],
                  "baseline_exp": ["session", "x", "params"], "attention_exp": ["session", "x", "params"],
                  "logarithm": ["session", "x", "params", "big_input_check"]},
    "nn": {"relu": ["session", "x"], "maxcut": ["session", "x", "cast_width", "eps_ulps"],
           "softmax_parts": ["session", "x", "params", "base2", "cast_width"],
           "softmax": ["session", "x", "params", "base2", "cast_width"],
           "attention_block": ["session", "heads", "params", "optimized", "cast_width"],
           "linear_layer": ["session", "x", "layer"], "mlp_forward": ["session", "x", "layers"]},
}


@pytest.mark.parametrize("mod", sorted(SIGNATURES))
def test_facade_signatures_are_the_references(mod):
    import importlib
    m = importlib.import_module(f"paper_2402_02320_b200.mpfix.{mod}")
    for name, params in SIGNATURES[mod].items():
        got = list(inspect.signature(getattr(m, name)).parameters)
        assert got == params, (mod, name, got)


def test_install_aliases_mpfix():
    from paper_2402_02320_b200 import mpfix
    saved = {k: v for k, v in sys.modules.items() if k == "mpfix" or k.startswith("mpfix.")}
    try:
        mpfix.install()
        import mpfix as alias
        from mpfix.protocols import mul
        from mpfix.session import PartySession
        from mpfix.transport import InProcHub, NullMesh  # noqa: F401
        assert alias is mpfix and mul is mpfix.protocols.mul and PartySession is mpfix.PartySession
        for nm in ("AShare", "BShare", "share_arith", "share_bits", "reconstruct_arith", "reconstruct_bits",
                   "PartySession", "CommMetrics", "OpCounters", "ApproxParams", "DEFAULT_PARAMS", "reciprocal",
                   "exponentiation", "logarithm", "baseline_exp", "attention_exp", "AttentionDims",
                   "LinearLayer", "relu", "maxcut", "softmax", "attention_block", "linear_layer",
                   "mlp_forward", "fold_base2"):
            assert hasattr(alias, nm), nm
    finally:
        for k in [k for k in sys.modules if k == "mpfix" or k.startswith("mpfix.")]:
            del sys.modules[k]
        sys.modules.update(saved)


@pytest.fixture(scope="module")
def facade():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from facade_engine import FacadeEngine
    return FacadeEngine()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case_through_facade(facade, name):
    fn, n = CASES[name]
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    info = json.loads(bytes(z["info"]).decode())
    got, ginfo = facade.run(fn, n)
    assert ginfo["demands"] == info["demands"]
    assert ginfo["total"] == info["total"]
    assert ginfo["ledger"] == info["ledger"]
    for k, v in got.items():
        want = z[f"out__{k}"]
        assert v.shape == want.shape, (k, v.shape, want.shape)
        assert np.array_equal(v, want), k


@pytest.mark.gpu
def test_facade_sharing_helpers_and_generate_material(facade):
    from paper_2402_02320_b200.mpfix import preprocessing as FP
    from paper_2402_02320_b200.mpfix import sharing as FS
    d = np.load(os.path.join(GOLDEN, "dealer.npz"))
    key = FP.triple_key(64)
    per = FP.generate_material(11, 3, key, 13)
    for nm in ("a", "b", "c"):
        assert np.array_equal(np.stack([per[p][nm] for p in range(3)]), d[f"{key.name()}__13__{nm}"])
    rng = np.random.default_rng(5)
    sec = rng.integers(0, 1 << 64, 50, dtype=np.uint64)
    sh = FS.share_arith(np.random.Generator(np.random.Philox(key=[7, 7])), sec, 4, 64)
    assert np.array_equal(FS.reconstruct_arith(sh), sec)
    bits = rng.integers(0, 2, (9, 8), dtype=np.uint8)
    bs = FS.share_bits(np.random.Generator(np.random.Philox(key=[8, 8])), bits, 3)
    assert np.array_equal(FS.reconstruct_bits(bs), bits)
    pa = FS.public_ashare(5, 64, 0, 0, shape=(3,))
    assert np.array_equal(pa.values, np.full(3, 5, np.uint64))
    assert np.array_equal(FS.public_ashare(5, 64, 0, 1, shape=(3,)).values, np.zeros(3, np.uint64))
    x = FS.AShare(np.arange(4, dtype=np.uint64), 64)
    assert np.array_equal(FS.add_public(x, np.uint64(3), 0).values, np.arange(4, dtype=np.uint64) + np.uint64(3))
    assert np.array_equal(FS.add_public(x, np.uint64(3), 2).values, np.arange(4, dtype=np.uint64))
    assert np.array_equal((x.mul_public(-1) + x).values, np.zeros(4, np.uint64))
    assert np.array_equal(x[1:3].values, np.array([1, 2], np.uint64))
