"""All-parties numpy simulation of the reference MPC engine (the CPU oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). Parity pinned by
``tests/test_oracle_golden.py`` against fixtures made from the reference.

Layout: every arithmetic share tensor is ``uint64[n_parties, *shape]`` masked
to the ring width; every binary share tensor is ``uint8[n_parties, *shape]``
(one byte per bit, trailing axis = bit index LSB first, as in the reference).
An opening is a sum (or XOR) over the leading party axis — the reference does
the same sum after an all-to-all broadcast (``session.py:87-115``). Because
the protocols are deterministic given inputs and dealer material, this
simulation produces every party's shares bit-for-bit as the reference does.

Each function names the reference ``file:line`` (relative to
``/root/reference/pkg/src/mpfix``) whose behaviour it restates.
"""

from __future__ import annotations

import hashlib
import math
from contextlib import contextmanager
from dataclasses import dataclass, field, fields

import numpy as np

U64 = np.uint64
_M64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# Philox4x64-10 byte stream  (numpy Generator.bytes; used by ring.py:124-134,
# preprocessing.py:121-125, scenarios.py:48-51, tests/helpers.py:55,72)

_PHILOX_M0 = 0xD2E7470EE14C6C93
_PHILOX_M1 = 0xCA5A826395121157
_PHILOX_W0 = 0x9E3779B97F4A7C15
_PHILOX_W1 = 0xBB67AE8584CAA73B


def _mulhilo(a: np.ndarray, m: int):
    """(hi, lo) of the 128-bit product a*m for uint64 array a, constant m."""
    lo32 = np.uint64(0xFFFFFFFF)
    a_lo, a_hi = a & lo32, a >> U64(32)
    m_lo, m_hi = U64(m & 0xFFFFFFFF), U64(m >> 32)
    ll, lh = a_lo * m_lo, a_lo * m_hi
    hl, hh = a_hi * m_lo, a_hi * m_hi
    mid = (ll >> U64(32)) + (lh & lo32) + (hl & lo32)
    lo = a * U64(m)
    hi = hh + (lh >> U64(32)) + (hl >> U64(32)) + (mid >> U64(32))
    return hi, lo


def philox4x64_blocks(key: tuple[int, int], first_block: int, nblocks: int) -> np.ndarray:
    """Philox4x64-10 output for counters first_block+1 .. (numpy pre-increments).

    Returns uint64[nblocks, 4]. Bit-exact with ``np.random.Philox`` raw output.
    """
    with np.errstate(over="ignore"):
        c0 = np.arange(first_block + 1, first_block + 1 + nblocks, dtype=U64)
        c1 = np.zeros(nblocks, U64)
        c2 = np.zeros(nblocks, U64)
        c3 = np.zeros(nblocks, U64)
        k0, k1 = key[0] & _M64, key[1] & _M64
        for _ in range(10):
            hi0, lo0 = _mulhilo(c0, _PHILOX_M0)
            hi1, lo1 = _mulhilo(c2, _PHILOX_M1)
            c0, c1, c2, c3 = hi1 ^ c1 ^ U64(k0), lo1, hi0 ^ c3 ^ U64(k1), lo0
            k0 = (k0 + _PHILOX_W0) & _M64
            k1 = (k1 + _PHILOX_W1) & _M64
    return np.stack([c0, c1, c2, c3], axis=1)


def philox_key(key) -> tuple[int, int]:
    """numpy's Philox(key=...) convention: an int is split into LE 64-bit words."""
    if isinstance(key, (int, np.integer)):
        k = int(key)
        return (k & _M64, (k >> 64) & _M64)
    words = [int(v) for v in np.asarray(key, dtype=U64).ravel()]
    words += [0] * (2 - len(words))
    return (words[0], words[1])


class ByteStream:
    """Restates ``Generator.bytes``: each call consumes ceil(L/4) 32-bit words
    from a contiguous u32 stream (low half of each u64 first); the unused
    tail bytes of the last word are dropped."""

    def __init__(self, key):
        self.key = philox_key(key)
        self.pos32 = 0

    def take(self, nbytes: int) -> np.ndarray:
        n32 = (nbytes + 3) // 4
        first_u64 = self.pos32 // 2
        last_u64 = (self.pos32 + n32 - 1) // 2
        b0, b1 = first_u64 // 4, last_u64 // 4
        raw = philox4x64_blocks(self.key, b0, b1 - b0 + 1).reshape(-1)
        words = raw.astype("<u8").view("<u4")
        start = self.pos32 - b0 * 8
        self.pos32 += n32
        return words[start:start + n32].view(np.uint8)[:nbytes].copy()

    def elems(self, shape, width: int) -> np.ndarray:       # ring.py:124-128
        n = int(np.prod(shape)) if shape else 1
        raw = self.take(8 * max(n, 1)).view("<u8").astype(U64)
        return wrap(raw[:n].reshape(shape), width)

    def bits(self, shape) -> np.ndarray:                     # ring.py:131-134
        n = int(np.prod(shape)) if shape else 1
        raw = self.take(max(n, 1))
        return (raw[:n] & np.uint8(1)).reshape(shape)


# ---------------------------------------------------------------------------
# Ring Z_2^w on uint64 (ring.py:20-121)


def mask(width: int) -> np.uint64:
    return U64(_M64 if width == 64 else (1 << width) - 1)


def wrap(v, width: int) -> np.ndarray:
    v = np.asarray(v, dtype=U64)
    return v if width == 64 else v & mask(width)


def to_ring(v, width: int) -> np.ndarray:                   # ring.py:35-41
    a = np.asarray(v)
    if a.dtype == U64:
        return wrap(a, width)
    return wrap(np.asarray(a, dtype=np.int64).view(U64), width)


def encode(x, width: int, frac: int) -> np.ndarray:         # ring.py:76-84
    scaled = np.floor(np.asarray(x, dtype=np.float64) * float(1 << frac))
    return to_ring(scaled.astype(np.int64), width)


def to_signed(v, width: int) -> np.ndarray:                 # ring.py:65-73
    v = wrap(v, width)
    if width == 64:
        return v.view(np.int64)
    out = v.astype(np.int64)
    return np.where(v & U64(1 << (width - 1)) != 0, out - np.int64(1 << width), out)


def decode(v, width: int, frac: int) -> np.ndarray:         # ring.py:87-89
    return to_signed(v, width).astype(np.float64) / float(1 << frac)


def bits_of(v, width: int) -> np.ndarray:                   # ring.py:110-114
    v = wrap(v, width)
    return ((v[..., None] >> np.arange(width, dtype=U64)) & U64(1)).astype(np.uint8)


def bits_to_uint(b, width: int) -> np.ndarray:              # ring.py:117-121
    b = np.asarray(b, dtype=U64)
    w = U64(1) << np.arange(b.shape[-1], dtype=U64)
    return wrap((b * w).sum(axis=-1, dtype=U64), width)


def rsum(a, width: int, axis=-1) -> np.ndarray:
    return wrap(np.asarray(a, U64).sum(axis=axis, dtype=U64), width)


# ---------------------------------------------------------------------------
# Share tensors with a party axis (sharing.py:21-121)


@dataclass
class AShare:
    values: np.ndarray  # uint64[n, *shape]
    width: int
    frac: int = 0

    @property
    def shape(self):
        return self.values.shape[1:]

    @property
    def size(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    def _like(self, v, frac=None):
        return AShare(wrap(v, self.width), self.width, self.frac if frac is None else frac)

    def __add__(self, o):
        if o.width != self.width:
            raise ValueError("width mismatch")
        return self._like(self.values + o.values)

    def __sub__(self, o):
        if o.width != self.width:
            raise ValueError("width mismatch")
        return self._like(self.values - o.values)

    def __neg__(self):
        return self._like(U64(0) - self.values)

    def mul_public(self, k, frac_delta: int = 0):             # sharing.py:47-50
        return self._like(self.values * to_ring(k, self.width), self.frac + frac_delta)

    def with_frac(self, f):
        return AShare(self.values, self.width, f)

    def copy(self):
        return AShare(self.values.copy(), self.width, self.frac)

    def last(self, idx):
        """Index the logical trailing axes (the party axis is kept)."""
        return AShare(self.values[(slice(None),) + _tup(idx)], self.width, self.frac)

    def reshape(self, shape):
        return AShare(self.values.reshape((self.values.shape[0],) + tuple(shape)), self.width, self.frac)


@dataclass
class BShare:
    bits: np.ndarray  # uint8[n, *shape]

    @property
    def shape(self):
        return self.bits.shape[1:]

    @property
    def size(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    def __xor__(self, o):
        return BShare(self.bits ^ o.bits)

    def last(self, idx):
        return BShare(self.bits[(slice(None),) + _tup(idx)])


def _tup(idx):
    return idx if isinstance(idx, tuple) else (idx,)


def add_public(x: AShare, const) -> AShare:                  # sharing.py:106-111
    out = x.values.copy()
    out[0] = wrap(out[0] + to_ring(const, x.width), x.width)
    return AShare(out, x.width, x.frac)


def xor_public(x: BShare, pub) -> BShare:                    # sharing.py:99-103
    out = x.bits.copy()
    out[0] = out[0] ^ np.asarray(pub, np.uint8)
    return BShare(out)


def public_ashare(n, const, width, frac, shape) -> AShare:   # sharing.py:114-121
    cv = np.broadcast_to(to_ring(const, width), shape)
    v = np.zeros((n,) + tuple(shape), U64)
    v[0] = cv
    return AShare(v, width, frac)


def share_arith_dealer(bs: ByteStream, secret, n, width) -> np.ndarray:
    """sharing.py:124-133: parties 0..n-2 draw, the LAST party gets the difference."""
    secret = wrap(secret, width)
    draws = [bs.elems(secret.shape, width) for _ in range(n - 1)]
    last = secret.copy()
    for d in draws:
        last = wrap(last - d, width)
    return np.stack(draws + [last])


def share_bits_dealer(bs: ByteStream, bits, n) -> np.ndarray:
    """sharing.py:144-152 (XOR analogue; last party gets the difference)."""
    bits = np.asarray(bits, np.uint8)
    draws = [bs.bits(bits.shape) for _ in range(n - 1)]
    last = bits.copy()
    for d in draws:
        last ^= d
    return np.stack(draws + [last])


def deal_inputs_arith(values, n, width, key) -> np.ndarray:
    """tests/helpers.py:52-61 / scenarios.py:54-64: FIRST party gets the difference."""
    enc = to_ring(np.asarray(values), width)
    bs = ByteStream(key)
    parts = [bs.elems(enc.shape, width) for _ in range(n - 1)]
    first = enc
    for p in parts:
        first = wrap(first - p, width)
    return np.stack([first] + parts)


def deal_inputs_bits(bits, n, key) -> np.ndarray:
    """tests/helpers.py:70-78."""
    arr = np.asarray(bits, np.uint8)
    bs = ByteStream(key)
    parts = [bs.bits(arr.shape) for _ in range(n - 1)]
    first = arr.copy()
    for p in parts:
        first ^= p
    return np.stack([first] + parts)


# ---------------------------------------------------------------------------
# Metrics (metrics.py:25-109) — one ledger; every party's counters are equal.


@dataclass
class Counters:
    mul_count: int = 0
    mul_elems: int = 0
    matmul_count: int = 0
    matmul_macs: int = 0
    and_count: int = 0
    and_elems: int = 0
    bit2a_elems: int = 0
    scale_count: int = 0
    trunc_count: int = 0
    open_count: int = 0
    rounds: int = 0
    bytes: int = 0

    def as_dict(self):
        return {f.name: getattr(self, f.name) for f in fields(self)}


class Ledger:
    def __init__(self, n_parties):
        self.n = n_parties
        self.total = Counters()
        self.by_scope: dict[str, Counters] = {}
        self._stack: list[str] = []

    @contextmanager
    def scope(self, name):
        self._stack.append(name)
        try:
            yield self
        finally:
            self._stack.pop()

    def count(self, **d):
        key = "/".join(self._stack) if self._stack else "(root)"
        e = self.by_scope.setdefault(key, Counters())
        for k, v in d.items():
            setattr(e, k, getattr(e, k) + v)
            setattr(self.total, k, getattr(self.total, k) + v)

    def scoped(self, prefix):
        out = Counters()
        for k, e in self.by_scope.items():
            if k == prefix or k.startswith(prefix + "/"):
                for f in fields(out):
                    setattr(out, f.name, getattr(out, f.name) + getattr(e, f.name))
        return out


# ---------------------------------------------------------------------------
# Trusted dealer (preprocessing.py:66-174) and the single-use store (:263-326)


def key_name(kind: str, width: int, params=()) -> str:       # preprocessing.py:71-80
    if kind == "bintriple":
        return "bintriple"
    if kind == "edabit":
        return f"edabit_w{width}_m{params[0]}"
    if kind == "mtriple":
        m, k, r = params
        return f"mtriple_w{width}_{m}x{k}x{r}"
    return f"{kind}_w{width}"


def parse_key(name: str):
    parts = name.split("_")
    kind = parts[0]
    if kind == "bintriple":
        return kind, 1, ()
    w = int(parts[1][1:])
    if kind == "edabit":
        return kind, w, (int(parts[2][1:]),)
    if kind == "mtriple":
        return kind, w, tuple(int(d) for d in parts[2].split("x"))
    return kind, w, ()


def dealer_key(seed: int, name: str) -> tuple[int, int]:     # preprocessing.py:121-125
    digest = hashlib.sha256(f"{seed}:{name}".encode()).digest()
    return philox_key(int.from_bytes(digest[:16], "little"))


def deal_material(seed: int, n: int, name: str, count: int) -> dict:
    """generate_material (preprocessing.py:128-174), party axis first."""
    kind, w, params = parse_key(name)
    bs = ByteStream(dealer_key(seed, name))
    if kind == "triple":
        a = bs.elems((count,), w)
        b = bs.elems((count,), w)
        c = wrap(a * b, w)
        return {"a": share_arith_dealer(bs, a, n, w), "b": share_arith_dealer(bs, b, n, w),
                "c": share_arith_dealer(bs, c, n, w)}
    if kind == "mtriple":
        m, k, r = params
        a = bs.elems((count, m, k), w)
        b = bs.elems((count, k, r), w)
        c = wrap(np.matmul(a, b), w)
        return {"a": share_arith_dealer(bs, a, n, w), "b": share_arith_dealer(bs, b, n, w),
                "c": share_arith_dealer(bs, c, n, w)}
    if kind == "bintriple":
        a = bs.bits((count,))
        b = bs.bits((count,))
        return {"a": share_bits_dealer(bs, a, n), "b": share_bits_dealer(bs, b, n),
                "c": share_bits_dealer(bs, a & b, n)}
    if kind == "dabit":
        r = bs.bits((count,))
        return {"arith": share_arith_dealer(bs, r.astype(U64), n, w),
                "bit": share_bits_dealer(bs, r, n)}
    if kind == "edabit":
        m = params[0]
        value = wrap(bs.elems((count,), w), m)
        arith = share_arith_dealer(bs, value, n, w)
        bits = share_bits_dealer(bs, bits_of(value, m), n)
        return {"arith": arith, "bits": bits}
    raise ValueError(kind)


class Exhausted(RuntimeError):
    pass


class Store:
    """MaterialStore with per-key monotone cursors (preprocessing.py:263-326)."""

    def __init__(self, seed: int, n: int, demands: dict[str, int]):
        self.n = n
        self._arr, self._count, self._cur = {}, {}, {}
        for name, count in demands.items():
            if count > 0:
                self._arr[name] = deal_material(seed, n, name, count)
                self._count[name] = count
                self._cur[name] = 0

    def _take(self, name, count):
        if name not in self._arr:
            raise Exhausted(f"no material of kind {name}")
        cur = self._cur[name]
        if cur + count > self._count[name]:
            raise Exhausted(f"{name} exhausted")
        self._cur[name] = cur + count
        return cur, self._arr[name]

    def triples(self, w, count):
        cur, a = self._take(key_name("triple", w), count)
        return tuple(a[k][:, cur:cur + count] for k in "abc")

    def mtriple(self, w, m, k, r):
        cur, a = self._take(key_name("mtriple", w, (m, k, r)), 1)
        return tuple(a[x][:, cur] for x in "abc")

    def bintriples(self, count):
        cur, a = self._take("bintriple", count)
        return tuple(a[k][:, cur:cur + count] for k in "abc")

    def dabits(self, w, count):
        cur, a = self._take(key_name("dabit", w), count)
        return a["arith"][:, cur:cur + count], a["bit"][:, cur:cur + count]

    def edabits(self, w, m, count):
        cur, a = self._take(key_name("edabit", w, (m,)), count)
        return a["arith"][:, cur:cur + count], a["bits"][:, cur:cur + count]

    def usage(self):
        return {k: {"consumed": self._cur[k], "available": self._count[k]} for k in sorted(self._count)}


class Demand:
    """DemandCounter (preprocessing.py:369-403): zero material, records demand."""

    def __init__(self, n):
        self.n = n
        self.demands: dict[str, int] = {}

    def _note(self, name, c):
        self.demands[name] = self.demands.get(name, 0) + c

    def triples(self, w, count):
        self._note(key_name("triple", w), count)
        z = np.zeros((self.n, count), U64)
        return z, z.copy(), z.copy()

    def mtriple(self, w, m, k, r):
        self._note(key_name("mtriple", w, (m, k, r)), 1)
        return (np.zeros((self.n, m, k), U64), np.zeros((self.n, k, r), U64),
                np.zeros((self.n, m, r), U64))

    def bintriples(self, count):
        self._note("bintriple", count)
        z = np.zeros((self.n, count), np.uint8)
        return z, z.copy(), z.copy()

    def dabits(self, w, count):
        self._note(key_name("dabit", w), count)
        return np.zeros((self.n, count), U64), np.zeros((self.n, count), np.uint8)

    def edabits(self, w, m, count):
        self._note(key_name("edabit", w, (m,)), count)
        return np.zeros((self.n, count), U64), np.zeros((self.n, count, m), np.uint8)


# ---------------------------------------------------------------------------
# Session: openings are reductions over the party axis (session.py:71-121)


class Sim:
    def __init__(self, n: int, store):
        self.n = n
        self.store = store
        self.ledger = Ledger(n)

    def scope(self, name):
        return self.ledger.scope(name)

    def open(self, items: list) -> list[np.ndarray]:
        """One round; payload = u4 per element for w<=32, u8 otherwise, bits packed."""
        nbytes = 0
        out = []
        for it in items:
            if isinstance(it, AShare):
                nbytes += it.size * (4 if it.width <= 32 else 8)
                out.append(rsum(it.values, it.width, axis=0))
            elif isinstance(it, BShare):
                nbytes += (it.size + 7) // 8
                out.append(np.bitwise_xor.reduce(it.bits, axis=0))
            else:
                raise TypeError(type(it))
        for _ in range(self.n - 1):
            self.ledger.count(bytes=nbytes)
        self.ledger.count(rounds=1, open_count=1)
        return out


# ---------------------------------------------------------------------------
# Basic protocols (protocols/basic.py)


def mul(s: Sim, x: AShare, y: AShare) -> AShare:             # basic.py:27-42
    if x.shape != y.shape:
        raise ValueError("shape mismatch")
    w = x.width
    a, b, c = (t.reshape((s.n,) + x.shape) for t in s.store.triples(w, x.size))
    d, e = s.open([AShare(wrap(x.values - a, w), w), AShare(wrap(y.values - b, w), w)])
    z = c + d * b + e * a
    z[0] += d * e
    s.ledger.count(mul_count=1, mul_elems=x.size)
    return AShare(wrap(z, w), w, x.frac + y.frac)


def batch_matmul(s: Sim, pairs) -> list[AShare]:             # basic.py:49-79
    trip, masked = [], []
    for x, y in pairs:
        if len(x.shape) != 2 or len(y.shape) != 2 or x.shape[1] != y.shape[0]:
            raise ValueError("bad matmul shapes")
        a, b, c = s.store.mtriple(x.width, x.shape[0], x.shape[1], y.shape[1])
        trip.append((a, b, c))
        masked += [AShare(wrap(x.values - a, x.width), x.width),
                   AShare(wrap(y.values - b, x.width), x.width)]
    opened = s.open(masked)
    out = []
    for i, (x, y) in enumerate(pairs):
        w = x.width
        a, b, c = trip[i]
        d, e = opened[2 * i], opened[2 * i + 1]
        z = c + np.matmul(d, b) + np.matmul(a, e)
        z[0] += np.matmul(d, e)
        s.ledger.count(matmul_count=1, matmul_macs=x.shape[0] * x.shape[1] * y.shape[1])
        out.append(AShare(wrap(z, w), w, x.frac + y.frac))
    return out


def matmul(s, x, y):
    return batch_matmul(s, [(x, y)])[0]


def and_gate(s: Sim, x: BShare, y: BShare) -> BShare:        # basic.py:82-95
    if x.shape != y.shape:
        raise ValueError("shape mismatch")
    a, b, c = (t.reshape((s.n,) + x.shape) for t in s.store.bintriples(x.size))
    d, e = s.open([BShare(x.bits ^ a), BShare(y.bits ^ b)])
    z = c ^ (d & b) ^ (e & a)
    z[0] ^= d & e
    s.ledger.count(and_count=1, and_elems=x.size)
    return BShare(z)


def carry_prefix(s: Sim, g: np.ndarray, p: np.ndarray) -> np.ndarray:   # basic.py:98-129
    m = g.shape[-1]
    sh = 1
    while sh < m:
        g_hi, p_hi, g_lo, p_lo = g[..., sh:], p[..., sh:], g[..., :-sh], p[..., :-sh]
        if sh * 2 >= m:
            z = and_gate(s, BShare(p_hi), BShare(g_lo)).bits
            g = np.concatenate([g[..., :sh], g_hi ^ z], axis=-1)
        else:
            z = and_gate(s, BShare(np.concatenate([p_hi, p_hi], -1)),
                         BShare(np.concatenate([g_lo, p_lo], -1))).bits
            cut = g_hi.shape[-1]
            g = np.concatenate([g[..., :sh], g_hi ^ z[..., :cut]], axis=-1)
            p = np.concatenate([p[..., :sh], z[..., cut:]], axis=-1)
        sh *= 2
    return g


def _sum_bits(p0: np.ndarray, carries: np.ndarray) -> BShare:         # basic.py:132-136
    shifted = np.concatenate([np.zeros_like(carries[..., :1]), carries[..., :-1]], -1)
    return BShare(p0 ^ shifted)


def public_add_bits(s: Sim, pub, x: BShare) -> BShare:                # basic.py:139-152
    pub = np.asarray(pub, np.uint8)
    if pub.shape != x.shape:
        raise ValueError("shape mismatch")
    g = x.bits & pub
    p = xor_public(x, pub).bits
    return _sum_bits(p.copy(), carry_prefix(s, g, p))


def binary_add(s: Sim, x: BShare, y: BShare) -> BShare:               # basic.py:155-161
    g = and_gate(s, x, y).bits
    p = x.bits ^ y.bits
    return _sum_bits(p.copy(), carry_prefix(s, g, p))


def bit2a(s: Sim, b: BShare, width: int) -> AShare:                   # basic.py:164-184
    r_a, r_b = s.store.dabits(width, b.size)
    r_a = r_a.reshape((s.n,) + b.shape)
    (c,) = s.open([BShare(b.bits ^ r_b.reshape((s.n,) + b.shape))])
    c64 = c.astype(U64)
    factor = wrap(U64(1) - (c64 + c64), width)
    z = r_a * factor
    z[0] += c64
    s.ledger.count(bit2a_elems=b.size)
    return AShare(wrap(z, width), width, 0)


def compose(s: Sim, bits: BShare, width: int, frac: int = 0) -> AShare:  # basic.py:187-196
    m = bits.shape[-1]
    ar = bit2a(s, bits, width)
    wts = wrap(U64(1) << np.arange(m, dtype=U64), width)
    return AShare(rsum(ar.values * wts, width), width, frac)


def decompose(s: Sim, x: AShare) -> BShare:                            # basic.py:199-214
    w = x.width
    r_a, r_b = s.store.edabits(w, w, x.size)
    r_a = r_a.reshape((s.n,) + x.shape)
    r_b = BShare(r_b.reshape((s.n,) + x.shape + (w,)))
    (c,) = s.open([AShare(wrap(x.values - r_a, w), w)])
    return public_add_bits(s, bits_of(c, w), r_b)


def gt(s: Sim, x: AShare, y: AShare) -> BShare:                        # basic.py:217-225
    d = y - x
    return decompose(s, d).last((Ellipsis, d.width - 1))


def const_share(s: Sim, value, width, frac, shape=()) -> AShare:        # basic.py:228-233
    enc = encode(np.broadcast_to(np.asarray(value, np.float64), shape), width, frac)
    v = np.zeros((s.n,) + tuple(np.shape(enc)), U64)
    v[0] = enc
    return AShare(v, width, frac)


def add_const(s: Sim, x: AShare, value: float) -> AShare:              # basic.py:236-239
    return add_public(x, encode(np.asarray([value]), x.width, x.frac)[0])


# ---------------------------------------------------------------------------
# Derived protocols (protocols/derived.py)


def _trunc_core(s: Sim, x: AShare, f: int) -> AShare:                  # derived.py:20-42
    w = x.width
    r_lo, _ = s.store.edabits(w, f, x.size)
    r_lo = AShare(r_lo.reshape((s.n,) + x.shape), w)
    hw = w - 1 - f
    if hw > 0:
        r_hi, _ = s.store.edabits(w, hw, x.size)
        r_hi = AShare(r_hi.reshape((s.n,) + x.shape), w)
    else:
        r_hi = AShare(np.zeros((s.n,) + x.shape, U64), w)
    masked = x + r_lo + r_hi.mul_public(U64(1) << U64(f))
    (c,) = s.open([masked])
    return AShare(add_public(-r_hi, wrap(c >> U64(f), w)).values, w, x.frac)


def unsigned_truncate(s: Sim, x: AShare, f: int, out_frac=None) -> AShare:   # derived.py:45-52
    if f == 0:
        return x.copy()
    z = _trunc_core(s, x, f)
    s.ledger.count(trunc_count=1)
    return z.with_frac(x.frac - f if out_frac is None else out_frac)


def truncate(s: Sim, x: AShare, f: int, out_frac=None) -> AShare:    # derived.py:55-70
    if f == 0:
        return x.copy()
    w = x.width
    z = _trunc_core(s, add_public(x, U64(1) << U64(w - 2)), f)
    z = add_public(z, U64((-(1 << (w - 2 - f))) & ((1 << w) - 1)))
    s.ledger.count(trunc_count=1)
    return z.with_frac(x.frac - f if out_frac is None else out_frac)


def scale_fixed(s: Sim, x: AShare, const: float, const_frac=None) -> AShare:  # derived.py:73-83
    cf = x.frac if const_frac is None else const_frac
    enc = encode(np.asarray([const]), x.width, cf)[0]
    s.ledger.count(scale_count=1)
    return AShare(wrap(x.values * enc, x.width), x.width, x.frac + cf)


def evaluate_poly(s: Sim, x: AShare, coeffs, frac: int) -> AShare:   # derived.py:86-108
    deg = len(coeffs) - 1
    pw = {1: x}
    for i in range(2, deg + 1):
        pw[i] = truncate(s, mul(s, pw[i - 1], x), frac)
    acc = None
    for i in range(1, deg + 1):
        if coeffs[i] == 0:
            continue
        t = scale_fixed(s, pw[i], coeffs[i], frac)
        acc = t if acc is None else acc + t
    if acc is None:
        acc = AShare(np.zeros(x.values.shape, U64), x.width, x.frac + frac)
    acc = add_const(s, acc, float(coeffs[0]))
    return truncate(s, acc, frac)


def evaluate_square_completed(s: Sim, x: AShare, lead_shift, t3, t2, lin, const, frac):  # derived.py:111-128
    u = add_const(s, x, t3)
    u2 = truncate(s, mul(s, u, u), frac)
    v = add_const(s, u2, t2)
    sq = mul(s, v, v)
    lead = truncate(s, sq, lead_shift, out_frac=sq.frac)
    lin_t = scale_fixed(s, x, lin, frac)
    acc = add_const(s, lead + lin_t, const)
    return truncate(s, acc, frac)


def lmo(s: Sim, bits: BShare) -> BShare:                               # derived.py:131-149
    m = bits.shape[-1]
    y = bits.bits.copy()
    sh = 1
    while sh < m:
        lo = y[..., :m - sh]
        hi = y[..., sh:]
        z = and_gate(s, BShare(lo.copy()), BShare(hi.copy())).bits
        y[..., :m - sh] = lo ^ hi ^ z
        sh *= 2
    above = np.concatenate([y[..., 1:], np.zeros_like(y[..., :1])], -1)
    return BShare(y ^ above)


def max_vec(s: Sim, x: AShare) -> AShare:                              # derived.py:152-170
    cur = x
    while cur.shape[-1] > 1:
        d = cur.shape[-1]
        h = d // 2
        u, v, rest = cur.last((Ellipsis, slice(0, h))), cur.last((Ellipsis, slice(h, 2 * h))), \
            cur.last((Ellipsis, slice(2 * h, None)))
        b = gt(s, u, v)
        sel = bit2a(s, b, x.width)
        win = v + mul(s, sel, u - v)
        cur = AShare(np.concatenate([win.values, rest.values], -1), x.width, x.frac)
    return cur.last((Ellipsis, 0))


# ---------------------------------------------------------------------------
# Non-linear functions (nonlinear.py)

LOG2_E = math.log2(math.e)
LN2 = math.log(2.0)
EXP2_COEFFS = (1.00000259, 0.69300383, 0.24144276, 0.05201146, 0.01353417)   # nonlinear.py:49
LOG2_COEFFS = (0.0, 1.442547, -0.726980, 0.496404, -0.268344)                # nonlinear.py:52
TAYLOR_EXP2 = tuple(LN2 ** k / math.factorial(k) for k in range(5))          # nonlinear.py:56


@dataclass(frozen=True)
class Square:                                                        # nonlinear.py:59-95
    lead_shift: int
    negative: bool
    t3: float
    t2: float
    t1: float
    t0: float

    @property
    def lead(self):
        v = 2.0 ** -self.lead_shift
        return -v if self.negative else v


EXP2_SQUARE = Square(6, False, 0.96074360, 6.15066406, 24.02000383, 23.85013773)
LOG2_SQUARE = Square(2, True, -0.46246981, 0.712932283, -0.366125013, -0.858977912)


@dataclass(frozen=True)
class Params:                                                        # nonlinear.py:98-108
    newton_iters: int = 5
    eps: float = 2.0 ** -14
    exp_coeffs: tuple = EXP2_COEFFS
    exp_square: Square = EXP2_SQUARE
    log_coeffs: tuple = LOG2_COEFFS
    log_square: Square = LOG2_SQUARE


DEFAULT = Params()


def _clog2(n):
    return max(1, (n - 1).bit_length())


def _compose_vals(vals: np.ndarray, width, frac) -> AShare:           # nonlinear.py:117-122
    wts = U64(1) << np.arange(vals.shape[-1], dtype=U64)
    return AShare(rsum(vals * wts, width), width, frac)


def _pow2_product(s: Sim, bits: list[AShare]) -> AShare:              # nonlinear.py:125-131
    out = None
    for i, b in enumerate(bits):
        f = add_public(b.mul_public((1 << (1 << i)) - 1), 1)
        out = f if out is None else mul(s, out, f)
    return out


def _newton_product(s: Sim, z: AShare, frac, iters) -> AShare:        # nonlinear.py:134-143
    q = add_const(s, -z, 1.0)
    acc = add_const(s, q, 1.0)
    for _ in range(1, iters):
        q = truncate(s, mul(s, q, q), frac)
        acc = truncate(s, mul(s, acc, add_const(s, q, 1.0)), frac)
    return acc


def reciprocal(s: Sim, x: AShare, params: Params = DEFAULT) -> AShare:   # nonlinear.py:146-176
    w, p = x.width, x.frac
    with s.scope("reciprocal"):
        bits = decompose(s, x)
        sign = bits.last((Ellipsis, w - 1))
        mag = BShare(bits.bits[..., :w - 1] ^ bits.bits[..., w - 1:w])
        sa = bit2a(s, sign, w)
        x_pos = x - mul(s, sa, x).mul_public(2)
        oh = lmo(s, mag)
        window = oh.bits[..., :2 * p][..., ::-1].copy()
        t = compose(s, BShare(window), w, frac=p)
        z = truncate(s, mul(s, t, x_pos), p)
        y = _newton_product(s, z, p, params.newton_iters)
        y = truncate(s, mul(s, t, y), p)
        return y - mul(s, sa, y).mul_public(2)


def exponentiation(s: Sim, x: AShare, params: Params = DEFAULT) -> AShare:  # nonlinear.py:179-213
    w, p = x.width, x.frac
    bias = min(p, 38 - p)
    with s.scope("exponentiation"):
        xp = scale_fixed(s, x, LOG2_E, p)
        xb = add_const(s, xp, float(bias))
        bits = decompose(s, xb)
        c = _clog2(w - p - 1)
        seg = np.concatenate([bits.bits[..., p:2 * p], bits.bits[..., 2 * p:2 * p + c],
                              bits.bits[..., w - 1:w]], -1)
        conv = bit2a(s, BShare(seg), w)
        t = _compose_vals(conv.values[..., :p], w, p)
        ints = [AShare(conv.values[..., p + i], w) for i in range(c)]
        pw = _pow2_product(s, ints)
        y = mul(s, pw, evaluate_poly(s, t, params.exp_coeffs, p))
        sg = add_public(-AShare(conv.values[..., p + c], w), 1)
        return truncate(s, mul(s, sg, y), bias, out_frac=p)


def logarithm(s: Sim, x: AShare, params: Params = DEFAULT, big_input_check=False) -> AShare:  # nonlinear.py:216-267
    w, p = x.width, x.frac
    with s.scope("logarithm"):
        if big_input_check:
            thr = const_share(s, 2.0 ** p - 2.0 ** -p, w, p, x.shape)
            big = bit2a(s, gt(s, x, thr), w)
            sh = unsigned_truncate(s, x, w - 2 * p, out_frac=p)
            x = x + mul(s, big, sh - x)
        bits = decompose(s, x)
        window = bits.last((Ellipsis, slice(0, 2 * p)))
        oh = lmo(s, window)
        below = np.concatenate([oh.bits[..., 1:], np.zeros_like(oh.bits[..., :1])], -1)
        paired = and_gate(s, window, BShare(below))
        r_bits = np.bitwise_xor.reduce(paired.bits, axis=-1)
        seg = np.concatenate([oh.bits, r_bits[..., None]], -1)
        conv = bit2a(s, BShare(seg), w)
        ohv = conv.values[..., :2 * p]
        r = AShare(conv.values[..., 2 * p], w)
        ew = to_ring(np.arange(2 * p, dtype=np.int64) - p, w)
        y_l = AShare(rsum(ohv * ew, w), w)
        mw = U64(1) << (U64(2 * p - 1) - np.arange(2 * p, dtype=U64))
        m = AShare(rsum(ohv * mw, w), w, p)
        doubled = x.mul_public(2) - mul(s, x, r)
        t = truncate(s, mul(s, doubled, m), p)
        t = add_const(s, t, -1.0)
        y_r = evaluate_poly(s, t, params.log_coeffs, p)
        pre = y_r + y_l.mul_public(1 << p, frac_delta=p) + r.mul_public(1 << p, frac_delta=p)
        y = truncate(s, scale_fixed(s, pre, LN2, p), p)
        if big_input_check:
            y = y + scale_fixed(s, big, (w - 2 * p) * LN2, p)
        return y


def baseline_exp(s: Sim, x: AShare, params: Params = DEFAULT) -> AShare:   # nonlinear.py:270-312
    w, p = x.width, x.frac
    le = 31
    with s.scope("baseline_exp"):
        xp = truncate(s, scale_fixed(s, x, LOG2_E, p), p)
        nar = AShare(wrap(xp.values, le), le, p)
        bits = decompose(s, nar)
        ge = encode(np.asarray([float(le - p - 1)]), le, p)[0]
        pub = np.broadcast_to(bits_of(ge, le), bits.shape).copy()
        gate = public_add_bits(s, pub, bits).bits[..., le - 1]
        c = _clog2(le - p)
        seg = np.concatenate([bits.bits[..., :p], bits.bits[..., p:p + c],
                              bits.bits[..., le - 1:le], gate[..., None]], -1)
        conv = bit2a(s, BShare(seg), w)
        t = _compose_vals(conv.values[..., :p], w, p)
        ints = [AShare(conv.values[..., p + i], w) for i in range(c)]
        pw = _pow2_product(s, ints)
        dp = evaluate_poly(s, t, TAYLOR_EXP2, p)
        y_pos = mul(s, pw, dp)
        y_neg = truncate(s, y_pos, 1 << c, out_frac=p)
        sg = AShare(conv.values[..., p + c], w)
        y = y_pos + mul(s, sg, y_neg - y_pos)
        keep = add_public(-AShare(conv.values[..., p + c + 1], w), 1)
        return mul(s, keep, y)


def attention_exp(s: Sim, x: AShare, params: Params = DEFAULT) -> AShare:  # nonlinear.py:315-356
    wi, p = x.width, x.frac
    wo = min(64, 2 * wi)
    sq = params.exp_square
    with s.scope("attention_exp"):
        delta = math.log2(params.exp_coeffs[4]) + sq.lead_shift
        xb = add_const(s, x, float(p) + delta)
        bits = decompose(s, xb)
        c = _clog2(p)
        seg = np.concatenate([bits.bits[..., :p], bits.bits[..., p:p + c],
                              bits.bits[..., wi - 1:wi]], -1)
        conv = bit2a(s, BShare(seg), wo)
        t = _compose_vals(conv.values[..., :p], wo, p)
        ints = [AShare(conv.values[..., p + i], wo) for i in range(c)]
        pw = _pow2_product(s, ints)
        ev = evaluate_square_completed(s, t, sq.lead_shift, sq.t3, sq.t2,
                                       sq.lead * sq.t1, sq.lead * sq.t0, p)
        y = mul(s, pw, ev)
        sg = add_public(-AShare(conv.values[..., p + c], wo), 1)
        return truncate(s, mul(s, sg, y), p, out_frac=p)


# ---------------------------------------------------------------------------
# NN ops (nn.py)


@dataclass(frozen=True)
class Linear:                                                        # nn.py:48-54
    weight: np.ndarray
    bias: np.ndarray | None = None


def narrow(x: AShare, width) -> AShare:                              # nn.py:68-74
    if width > x.width:
        raise ValueError("cannot widen")
    return AShare(wrap(x.values, width), width, x.frac)


def transpose(x: AShare) -> AShare:                                  # nn.py:77-79
    return AShare(np.ascontiguousarray(x.values.swapaxes(-1, -2)), x.width, x.frac)


def _bcast_last(r: AShare, d) -> AShare:                             # nn.py:87-89
    return AShare(np.ascontiguousarray(np.broadcast_to(r.values[..., None], r.values.shape + (d,))),
                  r.width, r.frac)


def relu(s: Sim, x: AShare) -> AShare:                               # nn.py:92-97
    zero = public_ashare(s.n, 0, x.width, x.frac, x.shape)
    return mul(s, bit2a(s, gt(s, x, zero), x.width), x)


def maxcut(s: Sim, x: AShare, cast_width=32, eps_ulps=1) -> AShare:  # nn.py:100-112
    if cast_width is not None and cast_width < x.width:
        x = narrow(x, cast_width)
    m = max_vec(s, x)
    return add_public(x - _bcast_last(m, x.shape[-1]), -eps_ulps)


def softmax_parts(s: Sim, x: AShare, params=DEFAULT, base2=False, cast_width=32):  # nn.py:115-136
    p = x.frac
    if not base2:
        with s.scope("rescale"):
            x = truncate(s, scale_fixed(s, x, LOG2_E), p)
    with s.scope("maxcut"):
        xm = maxcut(s, x, cast_width=cast_width)
    with s.scope("exp"):
        e = attention_exp(s, xm, params)
    with s.scope("sum_recip"):
        r = reciprocal(s, AShare(rsum(e.values, e.width), e.width, e.frac), params)
    return e, r


def softmax(s: Sim, x: AShare, params=DEFAULT, base2=False, cast_width=32) -> AShare:  # nn.py:139-147
    e, r = softmax_parts(s, x, params, base2, cast_width)
    with s.scope("normalize"):
        return truncate(s, mul(s, e, _bcast_last(r, e.shape[-1])), e.frac)


def _stack(xs) -> AShare:
    return AShare(np.stack([v.values for v in xs], axis=1), xs[0].width, xs[0].frac)


def attention_block(s: Sim, heads, params=DEFAULT, optimized=False, cast_width=32) -> AShare:  # nn.py:150-186
    if not heads:
        raise ValueError("need at least one head")
    p = heads[0][0].frac
    with s.scope("scores"):
        raw = batch_matmul(s, [(q, transpose(k)) for q, k, _ in heads])
        scores = truncate(s, _stack(raw), p)
    with s.scope("softmax"):
        e, r = softmax_parts(s, scores, params, base2=True, cast_width=cast_width)
    H = len(heads)
    if optimized:
        with s.scope("out_matmul"):
            ev = truncate(s, _stack(batch_matmul(s, [(e.last(h), heads[h][2]) for h in range(H)])), p)
        with s.scope("normalize"):
            return truncate(s, mul(s, ev, _bcast_last(r, ev.shape[-1])), p)
    with s.scope("normalize"):
        pm = truncate(s, mul(s, e, _bcast_last(r, e.shape[-1])), p)
    with s.scope("out_matmul"):
        return truncate(s, _stack(batch_matmul(s, [(pm.last(h), heads[h][2]) for h in range(H)])), p)


def linear_layer(s: Sim, x: AShare, layer: Linear) -> AShare:        # nn.py:189-196
    w, p = x.width, x.frac
    wq = encode(layer.weight, w, p)
    acc = AShare(wrap(np.matmul(x.values, wq), w), w, 2 * p)
    if layer.bias is not None:
        acc = add_public(acc, encode(layer.bias, w, 2 * p))
    return truncate(s, acc, p)


def mlp_forward(s: Sim, x: AShare, layers) -> AShare:                # nn.py:199-206
    for i, layer in enumerate(layers):
        with s.scope(f"layer{i}"):
            x = linear_layer(s, x, layer)
            if i + 1 < len(layers):
                x = relu(s, x)
    return x


# ---------------------------------------------------------------------------
# Harness helpers


def simulate(fn, n: int, seed: int = 11):
    """tests/helpers.py:17-49 restated: dry run for demand, deal, run once for
    all parties. Returns (result, session)."""
    dry = Sim(n, Demand(n))
    fn(dry)
    live = Sim(n, Store(seed, n, dry.store.demands))
    return fn(live), live


def opened(s: Sim, x: AShare) -> np.ndarray:
    return decode(s.open([x])[0], x.width, x.frac)


__all__ = [n for n in dir() if not n.startswith("_")] + ["_clog2"]
