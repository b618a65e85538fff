"""Additive and XOR share tensors resident in HBM (reference: sharing.py:21-159).

``AShare.values`` is ``int64[L, *shape]`` (uint64 words masked to the ring
width) holding the shares of the ``L`` parties this process hosts, in the
order of ``parties`` (sim mode: all n parties on one GPU; party mode: just
this rank's party). ``BShare`` is row-packed: ``words`` is ``int64[L, *rows]``
and, when ``axis`` is set, each word carries the ``m`` bits of the logical
trailing bit axis (LSB first), so a w-bit decomposition is one word per
element. Without ``axis`` each word holds a single bit (``m == 1``).

All arithmetic on shares runs in libmpx kernels; torch is used only for
allocation and layout (views, slicing, concatenation).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from . import kernels as K
from .ring import encode_scalar, to_ring_int

_M64 = (1 << 64) - 1


def _p0(parties) -> int:
    return parties.index(0) if 0 in parties else -1


def _empty_like(t: torch.Tensor, shape=None) -> torch.Tensor:
    return torch.empty(t.shape if shape is None else shape, dtype=torch.int64, device=t.device)


class AShare:
    """Additive shares in Z_2^width of one tensor, for the local parties."""

    __slots__ = ("values", "width", "frac", "parties")

    def __init__(self, values: torch.Tensor, width: int, frac: int = 0, parties=None):
        if values.dtype != torch.int64:
            raise TypeError("AShare values must be int64 words")
        if values.dim() < 1:
            raise ValueError("AShare values need a leading party axis")
        self.values = values if values.is_contiguous() else values.contiguous()
        self.width = int(width)
        self.frac = int(frac)
        self.parties = tuple(range(values.shape[0])) if parties is None else tuple(parties)
        if len(self.parties) != values.shape[0]:
            raise ValueError("party axis does not match `parties`")

    @classmethod
    def strided(cls, values: torch.Tensor, width: int, frac: int, parties) -> "AShare":
        """Non-contiguous view (e.g. a transpose) kept as is: only for operands
        that are read once by a stride-aware kernel (batch_matmul masks)."""
        out = cls.__new__(cls)
        out.values, out.width, out.frac, out.parties = values, int(width), int(frac), tuple(parties)
        return out

    # -- shape ---------------------------------------------------------------
    @property
    def shape(self):
        return tuple(self.values.shape[1:])

    @property
    def size(self) -> int:
        return math.prod(self.shape)

    @property
    def L(self) -> int:
        return self.values.shape[0]

    @property
    def p0(self) -> int:
        return _p0(self.parties)

    def _new(self, values, width=None, frac=None) -> "AShare":
        return AShare(values, self.width if width is None else width,
                      self.frac if frac is None else frac, self.parties)

    # -- local linear algebra (sharing.py:37-62) ---------------------------------
    def _lin(self, ka, other=None, kb=0, c0=0, cv=None, frac=None) -> "AShare":
        if other is not None:
            if other.width != self.width:
                raise ValueError(f"width mismatch: {self.width} vs {other.width}")
            if other.shape != self.shape:
                raise ValueError(f"shape mismatch: {self.shape} vs {other.shape}")
        out = _empty_like(self.values)
        K.ring_lin(out, self.values, ka, None if other is None else other.values, kb, c0, cv,
                   self.L, self.size, self.width, self.p0)
        return self._new(out, frac=frac)

    def __add__(self, other: "AShare") -> "AShare":
        return self._lin(1, other, 1)

    def __sub__(self, other: "AShare") -> "AShare":
        return self._lin(1, other, _M64)

    def __neg__(self) -> "AShare":
        return self._lin(_M64)

    def mul_public(self, k, frac_delta: int = 0) -> "AShare":
        """Multiply by a public integer (sharing.py:47-50). Local."""
        if isinstance(k, (np.ndarray, torch.Tensor)) and np.ndim(k) > 0:
            raise TypeError("mul_public takes a scalar; use ring ops for tensors")
        return self._lin(to_ring_int(int(k), self.width), frac=self.frac + frac_delta)

    def __getitem__(self, idx) -> "AShare":
        idx = idx if isinstance(idx, tuple) else (idx,)
        return self._new(self.values[(slice(None),) + idx].contiguous())

    def view_at(self, idx) -> "AShare":
        """Like ``self[idx]`` but a strided view (no copy): for operands read
        once by stride-aware kernels (batch_matmul masks)."""
        idx = idx if isinstance(idx, tuple) else (idx,)
        return AShare.strided(self.values[(slice(None),) + idx], self.width, self.frac, self.parties)

    def reshape(self, shape) -> "AShare":
        return self._new(self.values.reshape((self.L,) + tuple(shape)))

    def with_frac(self, frac: int) -> "AShare":
        return self._new(self.values, frac=frac)

    def copy(self) -> "AShare":
        return self._new(self.values.clone())

    def __repr__(self):
        return f"AShare(shape={self.shape}, width={self.width}, frac={self.frac}, parties={self.parties})"


def _split_index(idx, ndim: int):
    """Split a logical index into (leading-axes index, trailing-axis index)."""
    idx = idx if isinstance(idx, tuple) else (idx,)
    if any(i is Ellipsis for i in idx):
        e = idx.index(Ellipsis)
        fill = ndim - (len(idx) - 1)
        idx = idx[:e] + (slice(None),) * fill + idx[e + 1:]
    idx = idx + (slice(None),) * (ndim - len(idx))
    return idx[:-1], idx[-1]


class BShare:
    """XOR shares of a bit tensor for the local parties (row-packed words)."""

    __slots__ = ("words", "m", "axis", "parties")

    def __init__(self, words: torch.Tensor, m: int = 1, axis: bool = False, parties=None):
        if words.dtype != torch.int64:
            raise TypeError("BShare words must be int64")
        if not axis and m != 1:
            raise ValueError("per-bit layout has m == 1")
        if not 1 <= m <= 64:
            raise ValueError("at most 64 bits per row")
        self.words = words if words.is_contiguous() else words.contiguous()
        self.m = int(m)
        self.axis = bool(axis)
        self.parties = tuple(range(words.shape[0])) if parties is None else tuple(parties)

    @property
    def rows_shape(self):
        return tuple(self.words.shape[1:])

    @property
    def shape(self):
        return self.rows_shape + ((self.m,) if self.axis else ())

    @property
    def size(self) -> int:
        return math.prod(self.shape)

    @property
    def rows(self) -> int:
        return math.prod(self.rows_shape)

    @property
    def L(self) -> int:
        return self.words.shape[0]

    @property
    def p0(self) -> int:
        return _p0(self.parties)

    def _new(self, words, m=None, axis=None) -> "BShare":
        return BShare(words, self.m if m is None else m, self.axis if axis is None else axis, self.parties)

    # -- layout conversion -------------------------------------------------------
    def as_perbit(self) -> "BShare":
        """One bit per word, logical trailing axis moved into the word tensor."""
        if not self.axis:
            return self
        out = torch.empty((self.L * self.rows, self.m), dtype=torch.uint8, device=self.words.device)
        K.bits_unpack(out, self.words, self.L * self.rows, self.m)
        return BShare(out.to(torch.int64).view((self.L,) + self.shape), 1, False, self.parties)

    def as_rows(self) -> "BShare":
        """Pack a per-bit tensor's last axis (<= 64) into one word per row."""
        if self.axis:
            return self
        shp = self.rows_shape
        if len(shp) == 0 or shp[-1] > 64:
            raise ValueError(f"cannot pack a trailing axis of {shp[-1] if shp else 0} bits")
        m = shp[-1]
        rows = self.L * math.prod(shp[:-1])
        out = torch.empty((self.L,) + shp[:-1], dtype=torch.int64, device=self.words.device)
        K.bits_pack(out, self.words.to(torch.uint8), rows, m)
        return BShare(out, m, True, self.parties)

    def like_layout(self, other: "BShare") -> "BShare":
        if self.axis == other.axis and self.m == other.m and self.rows_shape == other.rows_shape:
            return self
        if self.shape != other.shape:
            raise ValueError(f"shape mismatch {self.shape} vs {other.shape}")
        return self.as_rows() if other.axis else self.as_perbit()

    # -- local ops -------------------------------------------------------------
    def __xor__(self, other: "BShare") -> "BShare":
        o = other.like_layout(self)
        out = torch.empty_like(self.words)
        K.bits_op(out, self.words, o.words, _lib.BITS_XOR, self.L, self.rows, self.m)
        return self._new(out)

    def and_public(self, pub_bits) -> "BShare":
        """AND with public bits; every party masks its share (sharing.py:84-86)."""
        pub = public_bits_words(pub_bits, self)
        out = torch.empty_like(self.words)
        K.bits_op(out, self.words, pub, _lib.BITS_AND_PUB, self.L, self.rows, self.m)
        return self._new(out)

    def gather(self, src, axis: bool = True) -> "BShare":
        """New trailing bit axis made of bits ``src`` of this one (-1 = zero)."""
        if not self.axis:
            raise ValueError("gather needs a packed bit axis")
        out = torch.empty_like(self.words)
        K.bits_gather(out, self.words, list(src), self.L * self.rows)
        if not axis:
            return BShare(out, 1, False, self.parties)
        return BShare(out, len(src), True, self.parties)

    def __getitem__(self, idx) -> "BShare":
        if not self.axis:
            idx = idx if isinstance(idx, tuple) else (idx,)
            return self._new(self.words[(slice(None),) + idx].contiguous())
        lead, last = _split_index(idx, len(self.shape))
        base = self if all(isinstance(i, slice) and i == slice(None) for i in lead) else \
            self._new(self.words[(slice(None),) + lead].contiguous())
        if isinstance(last, (int, np.integer)):
            k = int(last) % self.m
            return base.gather([k], axis=False)
        if isinstance(last, slice):
            src = list(range(self.m))[last]
            if src == list(range(self.m)):
                return base
            return base.gather(src)
        raise TypeError(f"unsupported bit index {last!r}")

    def copy(self) -> "BShare":
        return self._new(self.words.clone())

    @property
    def bits(self) -> torch.Tensor:
        """uint8 view of the shares, one byte per bit, ``[L, *shape]`` (compat)."""
        if not self.axis:
            return self.words.to(torch.uint8)
        out = torch.empty((self.L * self.rows, self.m), dtype=torch.uint8, device=self.words.device)
        K.bits_unpack(out, self.words, self.L * self.rows, self.m)
        return out.view((self.L,) + self.shape)

    def __repr__(self):
        return f"BShare(shape={self.shape}, m={self.m}, axis={self.axis}, parties={self.parties})"


# ---------------------------------------------------------------------------
# Public-constant helpers (sharing.py:99-121)


def public_bits_words(pub_bits, like: BShare) -> torch.Tensor:
    """Pack public bits shaped like ``like`` into its row-word layout (one row of words)."""
    if isinstance(pub_bits, torch.Tensor):
        arr = pub_bits.to("cpu").numpy()
    else:
        arr = np.asarray(pub_bits, dtype=np.uint8)
    if tuple(arr.shape) != like.shape:
        raise ValueError(f"shape mismatch {arr.shape} vs {like.shape}")
    dev = like.words.device
    if like.axis:
        w = (arr.astype(np.uint64) << np.arange(like.m, dtype=np.uint64)).sum(axis=-1, dtype=np.uint64)
    else:
        w = arr.astype(np.uint64)
    t = torch.from_numpy(np.ascontiguousarray(w).view(np.int64).reshape(like.rows_shape))
    return t.to(dev) if dev.type != "meta" else torch.empty(t.shape, dtype=torch.int64, device="meta")


def xor_public(x: BShare, pub_bits, party=None) -> BShare:
    """XOR a public bit pattern in; only party 0 flips (sharing.py:99-103)."""
    pub = public_bits_words(pub_bits, x)
    out = torch.empty_like(x.words)
    K.bits_op(out, x.words, pub, _lib.BITS_XOR_PUB, x.L, x.rows, x.m, x.p0)
    return x._new(out)


def _const_tensor(const, like: torch.Tensor, width: int):
    """Public ring constant(s) as (c0 scalar, cv device vector or None)."""
    if isinstance(const, torch.Tensor):
        return 0, const.to(device=like.device, dtype=torch.int64).reshape(-1)
    arr = np.asarray(const)
    if arr.ndim == 0:
        return to_ring_int(int(arr) if arr.dtype.kind in "iu" else arr.item(), width), None
    v = to_ring_np(arr, width).view(np.int64).reshape(-1)
    if like.device.type == "meta":
        return 0, torch.empty(v.shape, dtype=torch.int64, device="meta")
    return 0, torch.from_numpy(v.copy()).to(like.device)


def to_ring_np(arr, width):
    a = np.asarray(arr)
    if a.dtype != np.uint64:
        a = a.astype(np.int64).view(np.uint64)
    return a & np.uint64(_M64 if width == 64 else (1 << width) - 1)


def add_public(x: AShare, const, party=None) -> AShare:
    """Add a public ring constant (broadcast over trailing dims); party 0 only."""
    c0, cv = _const_tensor(const, x.values, x.width)
    out = _empty_like(x.values)
    K.ring_lin(out, x.values, 1, None, 0, c0, cv, x.L, x.size, x.width, x.p0)
    return x._new(out)


def public_ashare(const, width: int, frac: int, session, shape=None) -> AShare:
    """Degenerate sharing of a public value: party 0 holds it (sharing.py:114-121)."""
    shape = () if shape is None else tuple(shape)
    vals = session.alloc((session.L,) + shape)
    c0, cv = _const_tensor(const, vals, width)
    K.ring_lin(vals, None, 0, None, 0, c0, cv, session.L, math.prod(shape), width, session.p0)
    return AShare(vals, width, frac, session.parties)


def add_const(x: AShare, value: float) -> AShare:
    return add_public(x, encode_scalar(value, x.width, x.frac))
