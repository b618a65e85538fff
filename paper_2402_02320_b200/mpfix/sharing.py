"""``mpfix.sharing`` (sharing.py:21-159): one party's share tensors, resident in HBM.

``AShare(values, width, frac)`` and ``BShare(bits)`` take and expose numpy
arrays like the reference's dataclasses, but the words live in a CUDA tensor
and every local operation is a libmpx kernel. ``values`` / ``bits`` copy to
the host lazily (first access) and are cached; protocol calls pass the
device tensors straight to the engine.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .. import kernels as K
from .. import sharing as ES
from . import ring
from ._bridge import device, download_u64, upload_u64

_M64 = (1 << 64) - 1
_NOPARTY = (1,)   # local ops never place public constants: any non-zero party id


class AShare:
    """One party's additive share of a tensor over Z_2^width (sharing.py:21-62)."""

    __slots__ = ("_t", "_host", "width", "frac")

    def __init__(self, values, width: int, frac: int = 0):
        self.width = int(width)
        self.frac = int(frac)
        if isinstance(values, torch.Tensor):
            self._t, self._host = values, None
        else:
            arr = np.asarray(values, dtype=np.uint64)
            self._t, self._host = upload_u64(arr).reshape(arr.shape), None

    # -- engine bridge --------------------------------------------------------
    @classmethod
    def _from_engine(cls, s: ES.AShare) -> "AShare":
        if s.L != 1:
            raise ValueError("mpfix.AShare holds one party's share")
        return cls(s.values[0], s.width, s.frac)

    def _engine(self, parties=_NOPARTY) -> ES.AShare:
        t = self._t
        if t.dim() == 0:
            t = t.reshape(())
        return ES.AShare(t.unsqueeze(0), self.width, self.frac, parties)

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            self._host = np.zeros(self.shape, np.uint64) if self._t.is_meta else \
                download_u64(self._t).reshape(tuple(self._t.shape))
        return self._host

    @values.setter
    def values(self, arr):
        a = np.asarray(arr, dtype=np.uint64)
        self._t, self._host = upload_u64(a).reshape(a.shape), None

    @property
    def shape(self):
        return tuple(self._t.shape)

    @property
    def size(self) -> int:
        return int(math.prod(self.shape))

    # -- local linear algebra ---------------------------------------------------
    def _check_like(self, other):
        if not isinstance(other, AShare):
            raise TypeError(f"expected AShare, got {type(other).__name__}")
        if other.width != self.width:
            raise ValueError(f"width mismatch: {self.width} vs {other.width}")

    def __add__(self, other: "AShare") -> "AShare":
        self._check_like(other)
        return AShare._from_engine(self._engine() + other._engine())

    def __sub__(self, other: "AShare") -> "AShare":
        self._check_like(other)
        return AShare._from_engine(self._engine() - other._engine())

    def __neg__(self) -> "AShare":
        return AShare._from_engine(-self._engine())

    def mul_public(self, k, frac_delta: int = 0) -> "AShare":
        if np.ndim(k) == 0:
            return AShare._from_engine(self._engine().mul_public(int(k), frac_delta))
        kv = np.broadcast_to(ring.to_ring(k, self.width), self.shape)
        out = torch.empty_like(self._t)
        K.ring_mul(out, self._t, upload_u64(kv), self.size, self.width)
        return AShare(out, self.width, self.frac + frac_delta)

    def __getitem__(self, idx) -> "AShare":
        return AShare(self._t[idx].contiguous(), self.width, self.frac)

    def reshape(self, shape) -> "AShare":
        return AShare(self._t.reshape(shape), self.width, self.frac)

    def with_frac(self, frac: int) -> "AShare":
        return AShare(self._t, self.width, frac)

    def copy(self) -> "AShare":
        return AShare(self._t.clone(), self.width, self.frac)

    def __repr__(self):
        return f"AShare(shape={self.shape}, width={self.width}, frac={self.frac})"


class BShare:
    """One party's XOR share of a bit tensor (sharing.py:65-91)."""

    __slots__ = ("_e", "_host")

    def __init__(self, bits):
        if isinstance(bits, ES.BShare):
            self._e, self._host = bits, None
            return
        arr = np.asarray(bits, dtype=np.uint8)
        t = torch.from_numpy(np.ascontiguousarray(arr).astype(np.int64)).to(device())
        e = ES.BShare(t.unsqueeze(0), 1, False, _NOPARTY)
        if arr.ndim >= 1 and 0 < arr.shape[-1] <= 64:
            e = e.as_rows()
        self._e, self._host = e, None

    @classmethod
    def _from_engine(cls, e: ES.BShare) -> "BShare":
        if e.L != 1:
            raise ValueError("mpfix.BShare holds one party's share")
        return cls(e)

    def _engine(self, parties=_NOPARTY) -> ES.BShare:
        e = self._e
        return ES.BShare(e.words, e.m, e.axis, parties)

    @property
    def bits(self) -> np.ndarray:
        if self._host is None:
            self._host = np.zeros(self.shape, np.uint8) if self._e.words.is_meta else \
                self._e.bits[0].cpu().numpy()
        return self._host

    @property
    def shape(self):
        return self._e.shape

    @property
    def size(self) -> int:
        return self._e.size

    def __xor__(self, other: "BShare") -> "BShare":
        return BShare(self._engine() ^ other._engine())

    def __getitem__(self, idx) -> "BShare":
        return BShare(self._engine()[idx])

    def and_public(self, pub_bits) -> "BShare":
        return BShare(self._engine().and_public(np.asarray(pub_bits, dtype=np.uint8)))

    def copy(self) -> "BShare":
        return BShare(self._engine().copy())

    def __repr__(self):
        return f"BShare(shape={self.shape})"


def _check_like(a: AShare, b: AShare) -> None:
    if a.width != b.width:
        raise ValueError(f"width mismatch: {a.width} vs {b.width}")


def xor_public(x: BShare, pub_bits, party: int) -> BShare:
    """Only party 0 flips (sharing.py:99-103)."""
    return BShare(ES.xor_public(x._engine((party,)), np.asarray(pub_bits, dtype=np.uint8)))


def add_public(x: AShare, const, party: int) -> AShare:
    """Only party 0 adds (sharing.py:106-111)."""
    return AShare._from_engine(ES.add_public(x._engine((party,)), np.asarray(const)))


class _OneParty:
    """Minimal session stand-in for ``public_ashare`` (L = 1 at ``party``)."""

    def __init__(self, party):
        self.L, self.parties, self.device = 1, (party,), device()
        self.p0 = 0 if party == 0 else -1

    def alloc(self, shape):
        return torch.empty(tuple(shape), dtype=torch.int64, device=self.device)


def public_ashare(const, width: int, frac: int, party: int, shape=None) -> AShare:
    """Party 0 holds the public value, everyone else zero (sharing.py:114-121)."""
    cv = np.asarray(const)
    shp = cv.shape if shape is None else tuple(shape)
    return AShare._from_engine(ES.public_ashare(cv if cv.ndim else cv.item(), width, frac, _OneParty(party), shp))


def share_arith(rng: np.random.Generator, secret, n_parties: int, width: int, frac: int = 0) -> list[AShare]:
    """Dealer split (sharing.py:124-133): parties 0..n-2 draw, the last holds the difference."""
    sec = upload_u64(ring.wrap(np.asarray(secret, dtype=np.uint64), width))
    shape = tuple(np.shape(secret))
    n = sec.numel()
    draws = [upload_u64(ring.random_elems(rng, shape, width)).reshape(-1) for _ in range(n_parties - 1)]
    last = sec.reshape(-1).clone()
    for d in draws:
        K.ring_lin(last, last, 1, d, _M64, 0, None, 1, n, width, -1)
    return [AShare(t.reshape(shape), width, frac) for t in draws + [last]]


def reconstruct_arith(shares: list[AShare]) -> np.ndarray:
    st = torch.stack([s._t.reshape(-1) for s in shares])
    out = torch.empty(st.shape[1], dtype=torch.int64, device=st.device)
    K.open_sum(out, st, len(shares), st.shape[1], shares[0].width)
    return download_u64(out).reshape(shares[0].shape)


def share_bits(rng: np.random.Generator, bits, n_parties: int) -> list[BShare]:
    """Bits split (sharing.py:144-152): the last party holds the XOR difference."""
    arr = np.asarray(bits, dtype=np.uint8)
    draws = [ring.random_bits(rng, arr.shape) for _ in range(n_parties - 1)]
    shares = [BShare(d) for d in draws]
    last = BShare(arr)
    for s in shares:
        last = last ^ s
    return shares + [last]


def reconstruct_bits(shares: list[BShare]) -> np.ndarray:
    acc = shares[0]
    for s in shares[1:]:
        acc = acc ^ s
    return acc.bits.copy()


__all__ = ["AShare", "BShare", "xor_public", "add_public", "public_ashare", "share_arith",
           "reconstruct_arith", "share_bits", "reconstruct_bits"]
