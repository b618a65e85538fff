"""Pin the CPU oracle against fixtures generated from the reference itself.

Every party's output shares must match bit-for-bit, as must the dry-run
material demand and the op/communication ledger. Also pins the oracle's
Philox4x64-10 restatement against numpy and the dealer restatement against
the reference's ``generate_material`` (tests/golden/dealer.npz).
"""

import json
import os

import numpy as np
import pytest

import oracle as O
from cases import CASES
from engines import OracleEngine

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    outs = {k[5:]: z[k] for k in z.files if k.startswith("out__")}
    info = json.loads(bytes(z["info"]).decode())
    return outs, info, int(z["n"])


@pytest.fixture(scope="module")
def engine():
    return OracleEngine()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(engine, name):
    fn, n = CASES[name]
    want, info, gn = load_golden(name)
    assert gn == n
    got, ginfo = engine.run(fn, n)
    assert ginfo["demands"] == info["demands"]
    assert set(got) == set(want)
    for k in want:
        assert got[k].shape == want[k].shape, (k, got[k].shape, want[k].shape)
        assert np.array_equal(got[k], want[k]), k
    assert ginfo["total"] == info["total"]
    assert ginfo["ledger"] == info["ledger"]


@pytest.mark.parametrize("key", [0, 7, 12345, (1 << 127) + 99, [1003, 2], [2001, 5]])
def test_philox_restatement_matches_numpy(key):
    g = np.random.Generator(np.random.Philox(key=key))
    bs = O.ByteStream(key)
    for L in (5, 7, 8, 1, 33, 64, 3, 1000):
        assert bs.take(L).tobytes() == g.bytes(L)


def test_dealer_restatement_matches_reference_generate_material():
    z = np.load(os.path.join(GOLDEN, "dealer.npz"))
    groups = {}
    for k in z.files:
        name, count, arr = k.split("__")
        groups.setdefault((name, int(count)), {})[arr] = z[k]
    assert len(groups) == 10
    for (name, count), arrays in groups.items():
        got = O.deal_material(11, 3, name, count)
        for arr, want in arrays.items():
            assert np.array_equal(got[arr], want), (name, arr)
