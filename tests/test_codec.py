"""Fixed-point codec and public ring views and fold_base2 (a35)
against golden vectors produced by the reference itself
(``tests/golden/make_codec_golden.py``: ring.py:65-121, nn.py:58-65).

Edge cases: negatives, floor at exact multiples and just below, the range
limits +-2^(w-1-p), out-of-range magnitudes, +-inf and NaN (numpy's x86
float->int64 cast gives INT64_MIN, which the device codec reproduces), narrow
widths 8 / 31 / 32, every sign boundary, and SPEC.md:45's known answer
encode(7.7, p=14) = 126156.
CPU: the oracle's codec and the engine's fold_base2. GPU: the device kernels
(mpx_encode / mpx_decode / mpx_to_signed / mpx_bits_unpack through the
``mpfix.ring`` facade, and the session's share_fixed + open).
"""

import os
import warnings

import numpy as np
import pytest

import oracle as O

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "codec.npz"))
ENC_CASES = [(64, 23), (64, 14), (64, 0), (32, 14), (31, 16), (8, 3)]
WIDTHS = (64, 32, 31, 8)


def test_known_answer_spec_45():
    assert int(G["known_answer"][0]) == 126156
    assert int(O.encode(np.array([7.7]), 64, 14)[0]) == 126156


@pytest.mark.parametrize("w,p", ENC_CASES)
def test_oracle_encode_matches_reference(w, p):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert np.array_equal(O.encode(G["x"], w, p), G[f"enc_w{w}_p{p}"])


@pytest.mark.parametrize("w", WIDTHS)
def test_oracle_views_match_reference(w):
    words = G["words"]
    assert np.array_equal(O.to_signed(words, w), G[f"signed_w{w}"])
    assert np.array_equal(O.bits_of(words, w), G[f"bits_w{w}"])
    for p in (0, 14, 23):
        if p < w:
            assert np.array_equal(O.decode(words, w, p), G[f"dec_w{w}_p{p}"])


def test_fold_base2_matches_reference():
    from paper_2402_02320_b200.nn import LinearLayer, fold_base2
    f1 = fold_base2(LinearLayer(G["fold_W"], G["fold_b"]))
    f2 = fold_base2(LinearLayer(G["fold_W"], None))
    assert np.array_equal(f1.weight, G["fold_W_out"]) and np.array_equal(f1.bias, G["fold_b_out"])
    assert np.array_equal(f2.weight, G["fold_W_out_nobias"]) and f2.bias is None and bool(G["fold_nobias_is_none"])


@pytest.fixture()
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.gpu
@pytest.mark.parametrize("w,p", ENC_CASES)
def test_device_encode_matches_reference(gpu, w, p):
    from paper_2402_02320_b200.mpfix import ring
    got = ring.encode(G["x"], w, p)
    want = G[f"enc_w{w}_p{p}"]
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(G["x"][i], int(got[i]), int(want[i])) for i in bad[:5]]


@pytest.mark.gpu
@pytest.mark.parametrize("w", WIDTHS)
def test_device_views_match_reference(gpu, w):
    from paper_2402_02320_b200.mpfix import ring
    words = G["words"]
    assert np.array_equal(ring.to_signed(words, w), G[f"signed_w{w}"])
    assert np.array_equal(ring.bits_of(words, w), G[f"bits_w{w}"])
    assert np.array_equal(ring.wrap(words, w), G[f"wrap_w{w}"])
    assert np.array_equal(ring.bits_to_uint(G[f"bits_w{w}"], w), G[f"wrap_w{w}"])
    for p in (0, 14, 23):
        if p < w:
            assert np.array_equal(ring.decode(words, w, p), G[f"dec_w{w}_p{p}"])
    if w == 64:
        assert np.array_equal(ring.cast_down(words, 64, 32), G["cast_64_32"])
        with pytest.raises(ValueError):
            ring.cast_down(words, 32, 64)


@pytest.mark.gpu
def test_share_fixed_then_open_is_the_reference_encoding(gpu):
    from paper_2402_02320_b200.preprocessing import DemandCounter
    from paper_2402_02320_b200.session import SimSession
    finite = np.isfinite(G["x"]) & (np.abs(G["x"]) < 2.0 ** 40)
    xs = G["x"][finite]
    for n in (2, 3):
        s = SimSession(n, None)
        opened = s.open_arith(s.share_fixed(xs, 64, 23, [1000, 2]))
        assert np.array_equal(opened.cpu().numpy().view(np.uint64), G["enc_w64_p23"][finite])
    assert DemandCounter((0,), 2).dry
