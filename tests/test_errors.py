"""Error semantics of the drop-in boundary (SURVEY §8b "Errors").

The reference raises ValueError for shape / width mismatches
(protocols/basic.py:30,59,85,147; sharing.py:96; nn.py:71,162), TypeError for
opening a non-share (session.py:84) and PreprocessingExhausted when a store
runs dry (preprocessing.py:61,286-294; its test tests/test_preprocessing.py:78).
The engine raises the same types from the same calls. CPU tests use dry-run
sessions (meta tensors, no kernels) and host-side stores; the GPU tests run
live sessions and the reference-compatible facade.
"""

import numpy as np
import pytest
import torch

import paper_2402_02320_b200 as G
from paper_2402_02320_b200 import nn, protocols as P
from paper_2402_02320_b200.preprocessing import (DemandCounter, MaterialStore, PreprocessingExhausted,
                                                 triple_key)
from paper_2402_02320_b200.session import PartySession, SimSession


def _dry(n=2):
    return SimSession(n, DemandCounter(tuple(range(n)), n))


def _sh(s, shape, width=64, frac=0):
    return s.share_ring(np.zeros(shape, np.uint64), width, frac, [1000, 2])


def test_mul_shape_and_width_mismatch():
    s = _dry()
    with pytest.raises(ValueError, match="shape"):
        P.mul(s, _sh(s, (4,)), _sh(s, (5,)))
    with pytest.raises(ValueError, match="width"):
        P.mul(s, _sh(s, (4,), 64), _sh(s, (4,), 32))


def test_matmul_bad_shapes():
    s = _dry()
    with pytest.raises(ValueError, match="matmul"):
        P.batch_matmul(s, [(_sh(s, (3, 4)), _sh(s, (5, 2)))])


def test_and_gate_shape_mismatch():
    s = _dry()
    x = s.share_bits(np.zeros((6, 8), np.uint8), [2000, 5])
    y = s.share_bits(np.zeros((5, 8), np.uint8), [2001, 5])
    with pytest.raises(ValueError, match="shape"):
        P.and_gate(s, x, y)


def test_public_add_bits_shape_mismatch():
    s = _dry()
    x = s.share_bits(np.zeros((6, 8), np.uint8), [2000, 5])
    with pytest.raises(ValueError, match="shape"):
        P.public_add_bits(s, np.zeros((5, 8), np.uint8), x)


def test_share_add_width_mismatch():
    s = _dry()
    with pytest.raises(ValueError, match="width"):
        _sh(s, (4,), 64) + _sh(s, (4,), 32)


def test_narrow_cannot_widen_and_attention_needs_heads():
    s = _dry()
    with pytest.raises(ValueError, match="widen"):
        nn.narrow(_sh(s, (4,), 32), 64)
    with pytest.raises(ValueError, match="head"):
        nn.attention_block(s, [])


def test_open_non_share_is_type_error():
    s = _dry()
    with pytest.raises(TypeError):
        s.open_many([np.zeros(3, np.uint64)])


def test_store_exhaustion_and_missing_kind():
    """tests/test_preprocessing.py:78 of the reference: taking past the dealt
    count raises PreprocessingExhausted; a kind never dealt raises too."""
    st = MaterialStore((0,), 2, device="cpu")
    z = torch.zeros((1, 4), dtype=torch.int64)
    st.add_material(triple_key(64), 4, {"a": z, "b": z.clone(), "c": z.clone()})
    st.take_triples(64, 3)
    with pytest.raises(PreprocessingExhausted, match="exhausted"):
        st.take_triples(64, 2)
    st.take_triples(64, 1)
    assert st.usage() == {"triple_w64": {"consumed": 4, "available": 4}}
    with pytest.raises(PreprocessingExhausted, match="no material"):
        st.take_triples(32, 1)
    with pytest.raises(PreprocessingExhausted):
        st.take_dabits(64, 1)
    assert issubclass(PreprocessingExhausted, RuntimeError)


def test_party_session_without_communicator_refuses_live_store():
    st = MaterialStore((0,), 3, device="cpu")
    with pytest.raises(RuntimeError, match="communicator"):
        PartySession(0, 3, None, st, device=torch.device("cpu"))
    dry = PartySession(0, 3, None, DemandCounter((0,), 3))     # dry runs need no peers
    assert not dry.fused
    assert SimSession(3, None, device="cpu").fused


@pytest.mark.gpu
def test_live_run_past_dealt_material_raises():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2402_02320_b200.preprocessing import device_store
    c = DemandCounter((0, 1), 2)
    sd = SimSession(2, c)
    P.mul(sd, _sh(sd, (100,)), _sh(sd, (100,)))
    s = SimSession(2, device_store(11, 2, c.demands))
    x = s.share_ring(np.arange(100, dtype=np.uint64), 64, 0, [1000, 2])
    P.mul(s, x, x)
    with pytest.raises(PreprocessingExhausted):
        P.mul(s, x, x)
    with pytest.raises(PreprocessingExhausted):
        G.reciprocal(s, s.share_fixed(np.ones(8), 64, 23, [1000, 3]))


@pytest.mark.gpu
def test_reference_facade_raises_reference_types():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from mpfix_helpers import run_mpc
    from paper_2402_02320_b200.mpfix.protocols import mul
    from paper_2402_02320_b200.mpfix.sharing import AShare

    def fn(s):
        x = AShare(np.arange(4, dtype=np.uint64), 64)
        y = AShare(np.arange(4, dtype=np.uint64), 32)
        errs = []
        for call in (lambda: x + y, lambda: mul(s, x, y), lambda: mul(s, x, AShare(np.zeros(5, np.uint64), 64)),
                     lambda: s.open_many([x.values])):
            try:
                call()
            except (ValueError, TypeError) as e:
                errs.append(type(e).__name__)
        return errs

    for errs in run_mpc(fn, 2):
        assert errs == ["ValueError", "ValueError", "ValueError", "TypeError"]
