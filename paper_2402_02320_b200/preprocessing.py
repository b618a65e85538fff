"""Trusted-dealer preprocessing on the device: generation and single-use store.

Mirrors ``preprocessing.py`` of the reference (key names :66-80, generation
:121-174, store :263-332, demand counter :369-403) with one change of
medium: the dealer runs on the GPU. Every draw reproduces numpy's
Philox4x64-10 ``Generator.bytes`` stream bit for bit, so
the shares each party receives are identical to the reference dealer's for
the same seed and demand, but they are generated in place in HBM in the
layouts the protocol kernels read:

* arithmetic material: ``int64[L, count]`` (one row per local party);
* bit material (bintriples, daBit bits, edaBit bits): a flat packed bit
  stream per party, ``int64[L, ceil(count/64) + 2]`` (bit t = item t), read by
  kernels as unaligned bit fields at ``cursor + row * row_bits``.

edaBit bits are only generated for keys whose consumer needs them
(decomposition); truncation discards them in the reference too
(derived.py:29,33). Store cursors advance exactly as the reference's.
"""

from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass

import torch

from . import kernels as K

KIND_TRIPLE = 1
KIND_MATRIX_TRIPLE = 2
KIND_BIN_TRIPLE = 3
KIND_DABIT = 4
KIND_EDABIT = 5

_KIND_NAMES = {KIND_TRIPLE: "triple", KIND_MATRIX_TRIPLE: "mtriple", KIND_BIN_TRIPLE: "bintriple",
               KIND_DABIT: "dabit", KIND_EDABIT: "edabit"}
_NAME_KINDS = {v: k for k, v in _KIND_NAMES.items()}
_M64 = (1 << 64) - 1


# MPX_DEALER_LEGACY=1: the draw -> store -> share kernel chain instead of the
# fused per-kind kernels (A/B timing and cross-checks)
LEGACY_DEALER = os.environ.get("MPX_DEALER_LEGACY", "0") not in ("", "0")


class PreprocessingExhausted(RuntimeError):
    """A run asked for more dealer material than was generated (preprocessing.py:61)."""


@dataclass(frozen=True)
class MaterialKey:
    kind: int
    width: int
    params: tuple = ()

    def name(self) -> str:                       # preprocessing.py:71-80
        base = _KIND_NAMES[self.kind]
        if self.kind == KIND_BIN_TRIPLE:
            return base
        if self.kind == KIND_EDABIT:
            return f"{base}_w{self.width}_m{self.params[0]}"
        if self.kind == KIND_MATRIX_TRIPLE:
            m, k, r = self.params
            return f"{base}_w{self.width}_{m}x{k}x{r}"
        return f"{base}_w{self.width}"

    @staticmethod
    def from_name(name: str) -> "MaterialKey":   # preprocessing.py:82-94
        parts = name.split("_")
        kind = _NAME_KINDS[parts[0]]
        if kind == KIND_BIN_TRIPLE:
            return MaterialKey(kind, 1)
        width = int(parts[1][1:])
        if kind == KIND_EDABIT:
            return MaterialKey(kind, width, (int(parts[2][1:]),))
        if kind == KIND_MATRIX_TRIPLE:
            return MaterialKey(kind, width, tuple(int(d) for d in parts[2].split("x")))
        return MaterialKey(kind, width)


def triple_key(w):
    return MaterialKey(KIND_TRIPLE, w)


def mtriple_key(w, m, k, r):
    return MaterialKey(KIND_MATRIX_TRIPLE, w, (m, k, r))


def bintriple_key():
    return MaterialKey(KIND_BIN_TRIPLE, 1)


def dabit_key(w):
    return MaterialKey(KIND_DABIT, w)


def edabit_key(w, m):
    return MaterialKey(KIND_EDABIT, w, (m,))


def dealer_philox_key(seed: int, key: MaterialKey) -> tuple[int, int]:
    """sha256(f"{seed}:{name}")[:16] little-endian -> Philox key words (preprocessing.py:121-125)."""
    digest = hashlib.sha256(f"{seed}:{key.name()}".encode()).digest()
    k = int.from_bytes(digest[:16], "little")
    return (k & _M64, k >> 64)


def _words(nbits: int) -> int:
    return (nbits + 63) // 64 + 2   # +2 spare words: unaligned 2-word bit-field reads


# ---------------------------------------------------------------------------
# Material views handed to the protocol kernels


@dataclass
class ArithMat:
    """``int64[L, count]`` slice of one arithmetic material array (party stride ps)."""
    t: torch.Tensor

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def ps(self) -> int:
        return self.t.stride(0)


@dataclass
class BitMat:
    """Packed bit stream of one material array plus the cursor's bit offset."""
    words: torch.Tensor
    bit: int

    @property
    def ptr(self) -> int:
        return self.words.data_ptr()

    @property
    def ps(self) -> int:
        return self.words.stride(0)


@dataclass
class BitTriples:
    a: torch.Tensor
    b: torch.Tensor
    c: torch.Tensor
    bit: int

    @property
    def a_ptr(self):
        return self.a.data_ptr()

    @property
    def b_ptr(self):
        return self.b.data_ptr()

    @property
    def c_ptr(self):
        return self.c.data_ptr()

    @property
    def ps(self):
        return self.a.stride(0)


# ---------------------------------------------------------------------------
# Device dealer


class Dealer:
    """Generates one key's material for the local parties ``p_lo .. p_lo+L-1``.

    Draw order per kind follows preprocessing.py:139-171 exactly; ``q`` is the
    running u32 index into the key's Philox stream.
    """

    def __init__(self, seed: int, n_parties: int, p_lo: int, L: int, device, key_slots: dict | None = None):
        self.seed, self.n, self.p_lo, self.L = seed, n_parties, p_lo, L
        self.device = torch.device(device)
        self._out = None   # when set: write shares into these existing arrays
        self.key_slots = key_slots   # MaterialKey -> int64[2] device slot (keys read at launch)

    def _e(self, *shape):
        return torch.empty(shape, dtype=torch.int64, device=self.device)

    def _z(self, *shape):
        return torch.zeros(shape, dtype=torch.int64, device=self.device)

    def _dst(self, name, shape, zero=False):
        if self._out is not None and name in self._out:
            return self._out[name]
        return self._z(*shape) if zero else self._e(*shape)

    def _share_arith(self, secret, key, q, count, w, name=None):
        out = self._dst(name, (self.L, count))
        K.deal_share_arith(out, secret, key, q, count, self.n, self.p_lo, self.L, w)
        return out, q + (self.n - 1) * 2 * count

    def _share_bits(self, secret, key, q, count, name=None):
        out = self._dst(name, (self.L, _words(count)), zero=True)
        K.deal_share_bits(out, secret, key, q, count, self.n, self.p_lo, self.L)
        return out, q + (self.n - 1) * ((count + 3) // 4)

    def _elems(self, key, q, count, w):
        out = self._e(count)
        K.philox_elems(out, key, q, count, w)
        return out, q + 2 * count

    def _bits(self, key, q, count):
        out = self._z(_words(count))
        K.philox_bits(out, key, q, count)
        return out, q + (count + 3) // 4

    def generate(self, key: MaterialKey, count: int, need_bits: bool = True, out: dict | None = None) -> dict:
        """Deal ``count`` items of ``key``; with ``out`` (a previous result for
        the same key and count) the shares are written in place, keeping
        every device pointer stable (CUDA-graph replays)."""
        if out is not None:
            flat = {k: (v.view(self.L, -1) if k in ("a", "b", "c") and v.dim() > 2 else v) for k, v in out.items()}
            self._out = flat
        try:
            return self._generate(key, count, need_bits)
        finally:
            self._out = None

    def _generate(self, key: MaterialKey, count: int, need_bits: bool) -> dict:
        pk = self.key_slots[key] if self.key_slots is not None else dealer_philox_key(self.seed, key)
        if not LEGACY_DEALER:
            return self._generate_fused(key, count, need_bits, pk)
        w = key.width
        q = 0
        if key.kind == KIND_TRIPLE:                       # preprocessing.py:139-145
            a, q = self._elems(pk, q, count, w)
            b, q = self._elems(pk, q, count, w)
            c = self._e(count)
            K.ring_mul(c, a, b, count, w)
            sa, q = self._share_arith(a, pk, q, count, w, "a")
            sb, q = self._share_arith(b, pk, q, count, w, "b")
            sc, q = self._share_arith(c, pk, q, count, w, "c")
            return {"a": sa, "b": sb, "c": sc}
        if key.kind == KIND_MATRIX_TRIPLE:                # preprocessing.py:146-152
            m, k, r = key.params
            a, q = self._elems(pk, q, count * m * k, w)
            b, q = self._elems(pk, q, count * k * r, w)
            c = self._e(count * m * r)
            K.gemm(c, a, b, count, m, k, r, m * k, k * r, m * r, False, w)
            sa, q = self._share_arith(a, pk, q, count * m * k, w, "a")
            sb, q = self._share_arith(b, pk, q, count * k * r, w, "b")
            sc, q = self._share_arith(c, pk, q, count * m * r, w, "c")
            L = self.L
            return {"a": sa.view(L, count, m, k), "b": sb.view(L, count, k, r),
                    "c": sc.view(L, count, m, r)}
        if key.kind == KIND_BIN_TRIPLE:                   # preprocessing.py:153-159
            a, q = self._bits(pk, q, count)
            b, q = self._bits(pk, q, count)
            c = self._z(a.numel())
            K.bits_op(c, a, b, 1, 1, a.numel(), 64)      # AND
            sa, q = self._share_bits(a, pk, q, count, "a")
            sb, q = self._share_bits(b, pk, q, count, "b")
            sc, q = self._share_bits(c, pk, q, count, "c")
            return {"a": sa, "b": sb, "c": sc}
        if key.kind == KIND_DABIT:                        # preprocessing.py:160-164
            r, q = self._bits(pk, q, count)
            r_el = self._e(count)
            K.bits_flat_to_rows(r_el, r.data_ptr(), 0, count, 1)
            arith, q = self._share_arith(r_el, pk, q, count, w, "arith")
            bit, q = self._share_bits(r, pk, q, count, "bit")
            return {"arith": arith, "bit": bit}
        if key.kind == KIND_EDABIT:                       # preprocessing.py:165-170
            m = key.params[0]
            value, q = self._elems(pk, q, count, min(w, m))
            arith, q = self._share_arith(value, pk, q, count, w, "arith")
            res = {"arith": arith}
            if need_bits:
                flat = self._z(_words(count * m))
                K.bits_rows_to_flat(flat, value, count, m)
                res["bits"], q = self._share_bits(flat, pk, q, count * m, "bits")
            return res
        raise ValueError(f"unknown material kind {key.kind}")

    def _generate_fused(self, key: MaterialKey, count: int, need_bits: bool, pk) -> dict:
        """One fused launch per key (two for an edaBit with bits, three plus
        the A @ B GEMM for a matrix triple); same draw order and results as
        ``_generate``'s kernel chain (preprocessing.py:139-171)."""
        n, p_lo, L, w = self.n, self.p_lo, self.L, key.width
        if key.kind == KIND_TRIPLE:                       # preprocessing.py:139-145
            sa, sb, sc = (self._dst(x, (L, count)) for x in "abc")
            K.deal_triple(sa, sb, sc, pk, count, n, p_lo, L, w)
            return {"a": sa, "b": sb, "c": sc}
        if key.kind == KIND_MATRIX_TRIPLE:                # preprocessing.py:146-152
            m, k, r = key.params
            ca, cb, cc = count * m * k, count * k * r, count * m * r
            a, b = self._e(ca), self._e(cb)
            sa, sb, sc = self._dst("a", (L, ca)), self._dst("b", (L, cb)), self._dst("c", (L, cc))
            q0 = 2 * (ca + cb)                              # after the A and B draws
            K.deal_gen_arith(sa, a, pk, 0, q0, ca, n, p_lo, L, w, w)
            K.deal_gen_arith(sb, b, pk, 2 * ca, q0 + (n - 1) * 2 * ca, cb, n, p_lo, L, w, w)
            c = self._e(cc)
            K.gemm(c, a, b, count, m, k, r, m * k, k * r, m * r, False, w)
            K.deal_share_arith(sc, c, pk, q0 + (n - 1) * 2 * (ca + cb), cc, n, p_lo, L, w)
            return {"a": sa.view(L, count, m, k), "b": sb.view(L, count, k, r), "c": sc.view(L, count, m, r)}
        if key.kind == KIND_BIN_TRIPLE:                   # preprocessing.py:153-159
            sa, sb, sc = (self._dst(x, (L, _words(count)), zero=True) for x in "abc")
            K.deal_bintriple(sa, sb, sc, pk, count, n, p_lo, L)
            return {"a": sa, "b": sb, "c": sc}
        if key.kind == KIND_DABIT:                        # preprocessing.py:160-164
            arith = self._dst("arith", (L, count))
            bit = self._dst("bit", (L, _words(count)), zero=True)
            K.deal_dabit(arith, bit, pk, count, n, p_lo, L, w)
            return {"arith": arith, "bit": bit}
        if key.kind == KIND_EDABIT:                       # preprocessing.py:165-170
            m = key.params[0]
            arith = self._dst("arith", (L, count))
            K.deal_gen_arith(arith, None, pk, 0, 2 * count, count, n, p_lo, L, m, w)
            res = {"arith": arith}
            if need_bits:
                bits = self._dst("bits", (L, _words(count * m)), zero=True)
                K.deal_edabit_bits(bits, pk, 2 * count + (n - 1) * 2 * count, count, m, w, n, p_lo, L)
                res["bits"] = bits
            return res
        raise ValueError(f"unknown material kind {key.kind}")


# ---------------------------------------------------------------------------
# Stores


class MaterialStore:
    """One process's device-resident material for its local parties.

    Items are handed out in generation order and never twice; every key keeps
    a forward-only cursor (preprocessing.py:263-291).
    """

    dry = False

    def __init__(self, parties, n_parties: int, device="cuda"):
        self.parties = tuple(parties)
        self.n_parties = n_parties
        self.device = torch.device(device)
        self._arrays: dict[MaterialKey, dict] = {}
        self._counts: dict[MaterialKey, int] = {}
        self._cursors: dict[MaterialKey, int] = {}

    @property
    def L(self) -> int:
        return len(self.parties)

    def add_material(self, key: MaterialKey, count: int, arrays: dict) -> None:
        self._arrays[key] = arrays
        self._counts[key] = count
        self._cursors.setdefault(key, 0)

    def _take(self, key: MaterialKey, count: int):
        if key not in self._arrays:
            raise PreprocessingExhausted(f"parties {self.parties}: no material of kind {key.name()} available")
        cur = self._cursors[key]
        if cur + count > self._counts[key]:
            raise PreprocessingExhausted(
                f"parties {self.parties}: {key.name()} exhausted "
                f"(have {self._counts[key]}, cursor {cur}, need {count})")
        self._cursors[key] = cur + count
        return cur, self._arrays[key]

    # -- typed accessors (preprocessing.py:300-326) ---------------------------

    def take_triples(self, width, count):
        cur, a = self._take(triple_key(width), count)
        return tuple(ArithMat(a[k][:, cur:cur + count]) for k in "abc")

    def take_matrix_triple(self, width, m, k, r):
        cur, a = self._take(mtriple_key(width, m, k, r), 1)
        return a["a"][:, cur], a["b"][:, cur], a["c"][:, cur]

    def take_bin_triples(self, count):
        cur, a = self._take(bintriple_key(), count)
        return BitTriples(a["a"], a["b"], a["c"], cur)

    def take_dabits(self, width, count):
        cur, a = self._take(dabit_key(width), count)
        return ArithMat(a["arith"][:, cur:cur + count]), BitMat(a["bit"], cur)

    def take_edabits(self, width, m, count, need_bits: bool = True):
        cur, a = self._take(edabit_key(width, m), count)
        bits = None
        if need_bits:
            if "bits" not in a:
                raise PreprocessingExhausted(f"{edabit_key(width, m).name()}: bit shares were not generated")
            bits = BitMat(a["bits"], cur * m)
        return ArithMat(a["arith"][:, cur:cur + count]), bits

    def usage(self) -> dict:
        return {k.name(): {"consumed": self._cursors[k], "available": self._counts[k]}
                for k in sorted(self._counts, key=lambda k: k.name())}

    def rewind(self) -> None:
        """Reset every cursor (benchmark harness only: reuses material that a
        fresh dealer run would regenerate identically for the same demand)."""
        for k in self._cursors:
            self._cursors[k] = 0


class DemandCounter(MaterialStore):
    """Dry-run store: hands out meta tensors and records demand (preprocessing.py:369-403)."""

    dry = True

    def __init__(self, parties, n_parties: int):
        super().__init__(parties, n_parties, device="meta")
        self.demands: dict[MaterialKey, int] = {}
        self.needs_bits: dict[MaterialKey, bool] = {}

    def _note(self, key, count):
        self.demands[key] = self.demands.get(key, 0) + count

    def _m(self, *shape):
        return torch.empty(shape, dtype=torch.int64, device="meta")

    def take_triples(self, width, count):
        self._note(triple_key(width), count)
        return tuple(ArithMat(self._m(self.L, count)) for _ in range(3))

    def take_matrix_triple(self, width, m, k, r):
        self._note(mtriple_key(width, m, k, r), 1)
        return self._m(self.L, m, k), self._m(self.L, k, r), self._m(self.L, m, r)

    def take_bin_triples(self, count):
        self._note(bintriple_key(), count)
        z = self._m(self.L, 1)
        return BitTriples(z, z, z, 0)

    def take_dabits(self, width, count):
        self._note(dabit_key(width), count)
        return ArithMat(self._m(self.L, count)), BitMat(self._m(self.L, 1), 0)

    def take_edabits(self, width, m, count, need_bits: bool = True):
        key = edabit_key(width, m)
        self._note(key, count)
        self.needs_bits[key] = self.needs_bits.get(key, False) or need_bits
        return ArithMat(self._m(self.L, count)), (BitMat(self._m(self.L, 1), 0) if need_bits else None)


def stream_u32(key: MaterialKey, count: int, n_parties: int, need_bits: bool = True) -> int:
    """u32 words of the key's Philox stream one all-parties deal of ``count``
    items draws (SURVEY App. A4 draw sizes: random_elems = 8 bytes per
    element, random_bits = 1 byte per bit, each draw rounded up to whole u32,
    ring.py:124-134; n-1 share draws per secret, sharing.py:124-152)."""
    n = n_parties
    q = lambda nbytes: (nbytes + 3) // 4  # noqa: E731
    if count <= 0:
        return 0
    if key.kind == KIND_TRIPLE:
        return (2 + 3 * (n - 1)) * q(8 * count)
    if key.kind == KIND_MATRIX_TRIPLE:
        m, k, r = key.params
        return n * (q(8 * count * m * k) + q(8 * count * k * r)) + (n - 1) * q(8 * count * m * r)
    if key.kind == KIND_BIN_TRIPLE:
        return (2 + 3 * (n - 1)) * q(count)
    if key.kind == KIND_DABIT:
        return n * q(count) + (n - 1) * q(8 * count)
    if key.kind == KIND_EDABIT:
        return n * q(8 * count) + ((n - 1) * q(count * key.params[0]) if need_bits else 0)
    raise ValueError(f"unknown material kind {key.kind}")


def stream_blocks(demands: dict, n_parties: int, needs_bits: dict | None = None) -> int:
    """Philox4x64-10 blocks (32 bytes of stream) one re-deal of ``demands``
    generates: the dealer's algorithmic ALU work."""
    u32 = 0
    for key, count in demands.items():
        nb = True if needs_bits is None else needs_bits.get(key, key.kind != KIND_EDABIT)
        u32 += stream_u32(key, count, n_parties, nb)
    return (u32 + 7) // 8


def device_store(seed: int, n_parties: int, demands: dict, parties=None, device="cuda",
                 needs_bits: dict | None = None, into: MaterialStore | None = None) -> MaterialStore:
    """Deal every demanded key for the local ``parties`` (memory_stores,
    preprocessing.py:356-366). With ``into`` (a store dealt before for the same
    demand) fresh material is written into its arrays in place and its
    cursors are reset: every device pointer stays valid (CUDA graphs)."""
    parties = tuple(range(n_parties)) if parties is None else tuple(parties)
    if list(parties) != list(range(parties[0], parties[0] + len(parties))):
        raise ValueError("local parties must be contiguous")
    store = into if into is not None else MaterialStore(parties, n_parties, device)
    dealer = Dealer(seed, n_parties, parties[0], len(parties), device)
    for key, count in sorted(demands.items(), key=lambda kv: kv[0].name()):
        if count <= 0:
            continue
        nb = True if needs_bits is None else needs_bits.get(key, key.kind != KIND_EDABIT)
        if into is not None:
            dealer.generate(key, count, need_bits=nb, out=into._arrays[key])
        else:
            store.add_material(key, count, dealer.generate(key, count, need_bits=nb))
    if into is not None:
        into.rewind()
    return store


class DealerGraph:
    """A whole re-deal of ``store`` (every demanded key, in place) captured in
    ONE CUDA graph.

    The dealer kernels read their Philox keys from device slots, so a replay
    for a new seed is: hash the seed's per-key keys on the host
    (preprocessing.py:121-125), one small copy into the slots, one graph
    launch - the same material as ``device_store(seed, ..., into=store)``,
    bit for bit (tests/test_train.py), at device speed instead of ~100
    Python-issued launches.
    """

    def __init__(self, store: MaterialStore, demands: dict, needs_bits: dict | None, seed0: int):
        self.store = store
        self.n, self.parties, self.device = store.n_parties, store.parties, store.device
        self.keys = [k for k, c in sorted(demands.items(), key=lambda kv: kv[0].name()) if c > 0]
        self.counts = {k: demands[k] for k in self.keys}
        self.need = {k: (True if needs_bits is None else needs_bits.get(k, k.kind != KIND_EDABIT)) for k in self.keys}
        self.slots = torch.zeros((max(1, len(self.keys)), 2), dtype=torch.int64, device=self.device)
        self._host = torch.zeros(self.slots.shape, dtype=torch.int64).pin_memory()
        self._copied = torch.cuda.Event()   # the pinned key buffer is free again
        slot_of = {k: self.slots[i] for i, k in enumerate(self.keys)}
        self._dealer = Dealer(seed0, self.n, self.parties[0], len(self.parties), self.device, key_slots=slot_of)
        self._write(seed0)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            self._deal()                     # warm-up: first-use work outside the capture
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._deal()
        store.rewind()

    def _deal(self):
        for k in self.keys:
            self._dealer.generate(k, self.counts[k], need_bits=self.need[k], out=self.store._arrays[k])

    def _write(self, seed: int):
        import numpy as np
        words = np.zeros((self.slots.shape[0], 2), dtype=np.uint64)
        for i, k in enumerate(self.keys):
            words[i] = dealer_philox_key(seed, k)
        self._copied.synchronize()
        self._host.copy_(torch.from_numpy(words.view(np.int64)))
        self.slots.copy_(self._host, non_blocking=True)
        self._copied.record()

    def redeal(self, seed: int) -> MaterialStore:
        """Fresh material for ``seed`` in place; cursors reset."""
        self._write(seed)
        self.graph.replay()
        self.store.rewind()
        return self.store
