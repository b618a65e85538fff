"""CPU (no GPU): the B200 protocol code, run as a dry run on ``meta`` tensors,
must request exactly the reference's dealer material and record exactly the
reference's op/communication ledger for every golden case. This pins the
control flow, the per-key material order/counts and the metric contract
(criteria 5, 6, 8) without touching a GPU."""

import json
import os

import numpy as np
import pytest

from cases import CASES
from gpu_engine import GpuEngine

from paper_2402_02320_b200.session import demands_by_name

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def engine():
    return GpuEngine()


@pytest.mark.parametrize("name", sorted(CASES))
def test_dry_run_matches_reference(engine, name):
    fn, n = CASES[name]
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    info = json.loads(bytes(z["info"]).decode())
    from paper_2402_02320_b200.session import SimSession
    from paper_2402_02320_b200.preprocessing import DemandCounter
    counter = DemandCounter(tuple(range(n)), n)
    sess = SimSession(n, counter)
    out = fn(engine, sess)
    assert demands_by_name(counter) == info["demands"]
    assert sess.metrics.total.as_dict() == info["total"]
    assert {k: v.as_dict() for k, v in sorted(sess.metrics.ledger.items())} == info["ledger"]
    # logical output shapes match the reference's per-party shares
    for k, v in out.items():
        want = z[f"out__{k}"].shape[1:]
        assert tuple(v.shape) == tuple(want), (k, v.shape, want)
