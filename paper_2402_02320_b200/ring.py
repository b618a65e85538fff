"""Ring Z_2^w helpers (reference ring.py:20-134).

Share arithmetic runs in libmpx kernels (see ``sharing.py``); this module
holds the scalar/public-value helpers and the device fixed-point codec.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import kernels as K

WIDTH_64 = 64
WIDTH_32 = 32
_M64 = (1 << 64) - 1


def mask(width: int) -> int:
    return _M64 if width >= 64 else (1 << width) - 1


def to_ring_int(v: int, width: int) -> int:
    """Python int (possibly negative) -> Z_2^w representative (ring.py:35-41)."""
    return int(v) & mask(width)


def encode_scalar(x: float, width: int, frac: int) -> int:
    """floor(x * 2^frac) two's complement in Z_2^w (ring.py:76-100)."""
    scaled = math.floor(float(np.float64(x) * np.float64(float(1 << frac))))
    return to_ring_int(scaled, width)


def encode(x, width: int, frac: int, device="cuda") -> torch.Tensor:
    """Device fixed-point encode of a public float tensor (ring.py:76-84)."""
    t = torch.as_tensor(np.array(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x,
                        dtype=torch.float64)
    if torch.device(device).type == "meta":
        return torch.empty(t.shape, dtype=torch.int64, device="meta")
    t = t.to(device).contiguous()
    out = torch.empty(t.shape, dtype=torch.int64, device=t.device)
    K.encode(out, t, t.numel(), width, frac)
    return out


def decode(values: torch.Tensor, width: int, frac: int) -> torch.Tensor:
    """Device fixed-point decode of opened ring values (ring.py:87-89)."""
    v = values.contiguous()
    out = torch.empty(v.shape, dtype=torch.float64, device=v.device)
    K.decode(out, v, v.numel(), width, frac)
    return out


def bits_of_np(values, width: int) -> np.ndarray:
    """Public bit decomposition on host values (ring.py:110-114)."""
    v = np.asarray(values, dtype=np.uint64) & np.uint64(mask(width))
    return ((v[..., None] >> np.arange(width, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)


def to_signed_np(values, width: int) -> np.ndarray:
    v = np.asarray(values).view(np.uint64) if np.asarray(values).dtype == np.int64 else \
        np.asarray(values, dtype=np.uint64)
    v = v & np.uint64(mask(width))
    if width == 64:
        return v.view(np.int64)
    out = v.astype(np.int64)
    return np.where(v & np.uint64(1 << (width - 1)) != 0, out - np.int64(1 << width), out)
