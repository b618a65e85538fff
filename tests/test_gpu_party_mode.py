"""GPU: the party-mode path (one PartySession per party, L=1, unfused mask ->
exchange -> finish kernels, per-party dealer slices) on one GPU via host
rendezvous threads, bit-exact against the reference golden fixtures."""

import json
import os

import numpy as np
import pytest
import torch

from cases import CASES

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PARTY_CASES = ["mul_n3", "mul_w32", "batch_matmul", "and_xor", "bit2a", "decompose_compose",
               "decompose_w32", "binary_add_l8", "gt_n5", "trunc_f23", "unsigned_truncate", "lmo_l8",
               "max_vec", "reciprocal_n3", "exp_p14", "log", "attention_exp", "baseline_exp",
               "relu", "softmax", "attention_heads", "mlp", "log_big", "consts"]


@pytest.fixture(scope="module")
def engine():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from gpu_engine import GpuEngine
    return GpuEngine()


@pytest.mark.parametrize("name", PARTY_CASES)
def test_party_mode_bit_exact(engine, name):
    from gpu_engine import run_party_threads
    fn, n = CASES[name]
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    info = json.loads(bytes(z["info"]).decode())
    got, ginfo, sessions = run_party_threads(engine, fn, n)
    assert ginfo["total"] == info["total"]
    assert ginfo["ledger"] == info["ledger"]
    for k, v in got.items():
        want = z[f"out__{k}"]
        assert v.shape == want.shape, (k, v.shape, want.shape)
        assert np.array_equal(v, want), k
