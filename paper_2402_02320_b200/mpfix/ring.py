"""``mpfix.ring`` (ring.py:1-134) over the engine's device kernels.

Same names, arguments and numpy-in / numpy-out contract as the reference's
public-value helpers: every elementwise map runs as a libmpx kernel
(``mpx_ring_lin``, ``mpx_ring_mul``, ``mpx_to_signed``, ``mpx_encode``,
``mpx_decode``, ``mpx_bits_pack/unpack``) and ``matmul`` is the tcgen05 /
SIMT Z_2^64 GEMM (``mpx_gemm``). ``random_elems`` / ``random_bits`` draw from
the caller's numpy ``Generator`` exactly as the reference does (8 bytes per
element, 1 byte per bit), so sharing streams stay identical; ``fits`` is a
predicate on public floats.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import kernels as K
from ._bridge import device, download_u64, upload_u64

U64 = np.uint64
FULL_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)
WIDTH_64 = 64
WIDTH_32 = 32
_M64 = (1 << 64) - 1


def mask(width: int) -> np.uint64:
    return FULL_MASK if width == 64 else np.uint64((1 << width) - 1)


def _lin(a, ka, b, kb, width):
    """out = ka*a + kb*b mod 2^w on the device; numpy broadcasting first."""
    if b is None:
        arr = np.asarray(a)
        shape = arr.shape
        ta, tb = upload_u64(arr), None
    else:
        xa, xb = np.broadcast_arrays(np.asarray(a), np.asarray(b))
        shape = xa.shape
        ta, tb = upload_u64(xa), upload_u64(xb)
    out = torch.empty(ta.shape, dtype=torch.int64, device=ta.device)
    K.ring_lin(out, ta, ka, tb, kb, 0, None, 1, ta.numel(), width, -1)
    return download_u64(out).reshape(shape)


def _as_u64(values) -> np.ndarray:
    arr = np.asarray(values)
    if arr.dtype == U64:
        return arr
    return np.asarray(arr, dtype=np.int64).view(U64)


def wrap(values, width: int) -> np.ndarray:
    return _lin(np.asarray(values, dtype=U64), 1, None, 0, width)


def to_ring(values, width: int) -> np.ndarray:
    return _lin(_as_u64(values), 1, None, 0, width)


def add(a, b, width: int) -> np.ndarray:
    return _lin(np.asarray(a, U64), 1, np.asarray(b, U64), 1, width)


def sub(a, b, width: int) -> np.ndarray:
    return _lin(np.asarray(a, U64), 1, np.asarray(b, U64), _M64, width)


def neg(a, width: int) -> np.ndarray:
    return _lin(np.asarray(a, U64), _M64, None, 0, width)


def mul(a, b, width: int) -> np.ndarray:
    xa, xb = np.broadcast_arrays(np.asarray(a, U64), np.asarray(b, U64))
    ta, tb = upload_u64(xa), upload_u64(xb)
    out = torch.empty(ta.shape, dtype=torch.int64, device=ta.device)
    K.ring_mul(out, ta, tb, ta.numel(), width)
    return download_u64(out).reshape(xa.shape)


def matmul(a, b, width: int) -> np.ndarray:
    """Z_2^w matrix product (ring.py:60-62) on the Z_2^64 GEMM kernels
    (batched over equal or broadcast leading dims)."""
    A, B = np.asarray(a, U64), np.asarray(b, U64)
    if A.ndim < 2 or B.ndim < 2:
        return wrap(np.matmul(A, B), width) if A.size == 0 or B.size == 0 else _vec_matmul(A, B, width)
    M, Kd = A.shape[-2:]
    Kb, N = B.shape[-2:]
    if Kd != Kb:
        raise ValueError(f"matmul: shapes {A.shape} and {B.shape} not aligned")
    lead = np.broadcast_shapes(A.shape[:-2], B.shape[:-2])
    A = np.broadcast_to(A, lead + (M, Kd))
    B = np.broadcast_to(B, lead + (Kd, N))
    batch = int(np.prod(lead)) if lead else 1
    out = torch.empty((batch, M, N), dtype=torch.int64, device=device())
    if batch and M and N:
        if Kd == 0:
            out.zero_()
        else:
            K.gemm(out, upload_u64(A), upload_u64(B), batch, M, Kd, N, M * Kd, Kd * N, M * N, False, width)
    return download_u64(out).reshape(lead + (M, N))


def _vec_matmul(A, B, width):
    a2 = A.reshape(1, -1) if A.ndim == 1 else A
    b2 = B.reshape(-1, 1) if B.ndim == 1 else B
    r = matmul(a2, b2, width)
    if A.ndim == 1:
        r = r[..., 0, :]
    if B.ndim == 1:
        r = r[..., 0]
    return r


def to_signed(values, width: int) -> np.ndarray:
    arr = np.asarray(values, dtype=U64)
    t = upload_u64(arr)
    out = torch.empty_like(t)
    K.to_signed(out, t, t.numel(), width)
    return download_u64(out).view(np.int64).reshape(arr.shape)


def encode(x, width: int, frac: int) -> np.ndarray:
    arr = np.asarray(x, dtype=np.float64)
    t = torch.from_numpy(np.ascontiguousarray(arr).copy()).to(device())
    out = torch.empty(t.shape, dtype=torch.int64, device=t.device)
    K.encode(out, t, t.numel(), width, frac)
    return download_u64(out).reshape(arr.shape)


def decode(values, width: int, frac: int) -> np.ndarray:
    arr = np.asarray(values, dtype=U64)
    t = upload_u64(arr)
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    K.decode(out, t, t.numel(), width, frac)
    return out.cpu().numpy().reshape(arr.shape)


def encode_scalar(x: float, width: int, frac: int) -> np.uint64:
    return U64(encode(np.asarray([x]), width, frac)[0])


def fits(x, width: int, frac: int) -> bool:
    lim = float(1 << (width - 1 - frac))
    arr = np.asarray(x, dtype=np.float64)
    return bool(np.all(arr >= -lim) and np.all(arr < lim))


def cast_down(values, width_from: int, width_to: int) -> np.ndarray:
    if width_to > width_from:
        raise ValueError("cast_down cannot widen")
    return wrap(values, width_to)


def bits_of(values, width: int) -> np.ndarray:
    arr = np.asarray(values, U64)
    t = upload_u64(arr)
    n = t.numel()
    if width < 64:
        K.ring_lin(t, t, 1, None, 0, 0, None, 1, n, width, -1)
    out = torch.empty((n, width), dtype=torch.uint8, device=t.device)
    K.bits_unpack(out, t, n, width)
    return out.cpu().numpy().reshape(arr.shape + (width,))


def bits_to_uint(bits, width: int) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint8)
    m = b.shape[-1]
    if m > 64:
        raise ValueError("bits_to_uint: at most 64 bits per value")
    rows = int(np.prod(b.shape[:-1])) if b.ndim > 1 else 1
    tb = torch.from_numpy(np.ascontiguousarray(b & 1).copy()).to(device())
    out = torch.empty((rows,), dtype=torch.int64, device=tb.device)
    K.bits_pack(out, tb, rows, m)
    if width < 64:
        K.ring_lin(out, out, 1, None, 0, 0, None, 1, rows, width, -1)
    return download_u64(out).reshape(b.shape[:-1])


def random_elems(rng: np.random.Generator, shape, width: int) -> np.ndarray:
    n = int(np.prod(shape)) if shape else 1
    raw = np.frombuffer(rng.bytes(8 * max(n, 1)), dtype="<u8").copy()
    return wrap(raw.reshape(shape), width)


def random_bits(rng: np.random.Generator, shape) -> np.ndarray:
    n = int(np.prod(shape)) if shape else 1
    raw = np.frombuffer(rng.bytes(max(n, 1)), dtype=np.uint8).copy()
    return (raw & np.uint8(1)).reshape(shape)
