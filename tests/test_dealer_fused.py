"""Fused per-kind dealer kernels (mpx_deal_triple / _gen_arith / _bintriple /
_dabit / _edabit_bits) vs the CPU restatement of the reference dealer
(oracle.deal_material = preprocessing.py:128-174, pinned to the reference's
own generate_material output in tests/test_oracle_golden.py).

Bit-exact for every kind at counts that are aligned and unaligned to the
Philox block (4 elements / 32 bit-bytes), at n = 2..5 parties, for the
all-parties (sim) dealer and for every party-subset dealer (party mode: a
rank deals only its own parties' shares), and with the key read from a
device slot (the dealer's CUDA graph)."""
import numpy as np
import pytest
import torch

import oracle as O


KINDS = ["triple_w64", "triple_w32", "mtriple_w64_3x5x2", "mtriple_w64_7x9x4", "bintriple", "dabit_w64",
         "dabit_w32", "edabit_w64_m64", "edabit_w64_m23", "edabit_w32_m32", "edabit_w64_m40", "edabit_w64_m2",
         "edabit_w64_m61", "edabit_w64_m1"]
COUNTS = [1, 3, 4, 13, 64, 67, 1000, 4099]


def _as_np(arr, want):
    g = arr.cpu().numpy()
    if want.dtype == np.uint8:          # packed bit stream -> one byte per bit
        flat = np.unpackbits(g.view(np.uint8), axis=-1, bitorder="little")
        return flat[:, :want[0].size].reshape(want.shape)
    return g.view(np.uint64).reshape(want.shape)


def _check(key_name, count, n, p_lo, L, slot=False, seed=11):
    from paper_2402_02320_b200.preprocessing import Dealer, MaterialKey, dealer_philox_key
    key = MaterialKey.from_name(key_name)
    if key.kind == "mtriple" and count > 67:
        count = 67
    slots = None
    if slot:
        k0, k1 = dealer_philox_key(seed, key)
        t = torch.tensor([k0 - (1 << 64) if k0 >= 1 << 63 else k0, k1 - (1 << 64) if k1 >= 1 << 63 else k1],
                         dtype=torch.int64, device="cuda")
        slots = {key: t}
    d = Dealer(seed if not slot else 0, n, p_lo, L, "cuda", key_slots=slots)
    got = d.generate(key, count, need_bits=True)
    want = O.deal_material(seed, n, key_name, count)
    for arr, w in want.items():
        assert np.array_equal(_as_np(got[arr], w[p_lo:p_lo + L]), w[p_lo:p_lo + L]), (key_name, count, n, p_lo, L, arr)


@pytest.mark.gpu
@pytest.mark.parametrize("key_name", KINDS)
@pytest.mark.parametrize("count", COUNTS)
def test_fused_dealer_all_parties(key_name, count):
    _check(key_name, count, 3, 0, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("key_name", ["triple_w64", "bintriple", "dabit_w64", "edabit_w64_m64", "edabit_w64_m23",
                                      "mtriple_w64_3x5x2"])
@pytest.mark.parametrize("n", [2, 4, 5])
def test_fused_dealer_party_subsets(key_name, n):
    for p_lo in range(n):
        for L in range(1, n - p_lo + 1):
            _check(key_name, 67, n, p_lo, L)


@pytest.mark.gpu
@pytest.mark.parametrize("key_name", ["triple_w64", "bintriple", "dabit_w32", "edabit_w64_m64", "mtriple_w64_7x9x4"])
def test_fused_dealer_device_key_slot(key_name):
    _check(key_name, 1000, 3, 0, 3, slot=True)


@pytest.mark.gpu
def test_fused_dealer_equals_legacy_chain_large():
    """At a LeNet-sized count the fused kernels reproduce the legacy
    draw -> store -> share chain word for word (n = 3)."""
    import paper_2402_02320_b200.preprocessing as P
    from paper_2402_02320_b200.preprocessing import Dealer, MaterialKey
    for name, count in [("bintriple", 1_000_003), ("triple_w64", 100_001), ("edabit_w64_m64", 50_001),
                        ("edabit_w64_m23", 100_003), ("dabit_w64", 70_001)]:
        key = MaterialKey.from_name(name)
        fused = Dealer(7, 3, 0, 3, "cuda").generate(key, count)
        P.LEGACY_DEALER = True
        try:
            legacy = Dealer(7, 3, 0, 3, "cuda").generate(key, count)
        finally:
            P.LEGACY_DEALER = False
        for k in fused:
            assert torch.equal(fused[k], legacy[k]), (name, k)


@pytest.mark.parametrize("n", [2, 3, 5])
def test_stream_accounting_matches_oracle_draws(n, monkeypatch):
    """preprocessing.stream_u32 (the dealer roofline's work count) equals the
    u32 words the restated reference dealer actually draws."""
    from paper_2402_02320_b200.preprocessing import MaterialKey, stream_u32
    used = {}
    orig = O.ByteStream.take

    def take(self, nbytes):
        used[id(self)] = used.get(id(self), 0) + (nbytes + 3) // 4
        return orig(self, nbytes)
    monkeypatch.setattr(O.ByteStream, "take", take)
    for name in ["triple_w64", "mtriple_w64_3x5x2", "bintriple", "dabit_w32", "edabit_w64_m23", "edabit_w32_m32"]:
        for count in (1, 13, 66):
            used.clear()
            O.deal_material(11, n, name, count)
            assert sum(used.values()) == stream_u32(MaterialKey.from_name(name), count, n, True), (name, count)
