"""Conversion between the reference's one-party share objects and the engine's.

The reference (``/root/reference/pkg/src/mpfix``) hands every party its own
``AShare(values: np.uint64[...], width, frac)`` / ``BShare(bits: np.uint8)``
(sharing.py:21-91) and runs one ``PartySession`` per party thread or
process. The engine keeps shares in HBM with a leading local-party axis
(``paper_2402_02320_b200.sharing``). This module keeps the reference's
objects as thin handles over device tensors:

* an ``mpfix.AShare`` holds an ``int64[*shape]`` CUDA tensor; ``.values``
  copies it to the host on first access (the reference's numpy view), so a
  chain of protocol calls never leaves HBM;
* ``to_engine(obj, session)`` rebinds handles (recursively through lists
  and tuples) to engine shares of the session's party (L = 1) without copies;
* ``from_engine(obj)`` wraps engine results back into handles.

The product path is the engine's CUDA kernels; nothing here computes on
share values on the host.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import sharing as ES


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("mpfix (B200 engine) needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def upload_u64(arr) -> torch.Tensor:
    """numpy ring words (any integer dtype) -> contiguous int64 CUDA tensor (bit copy)."""
    a = np.asarray(arr)
    if a.dtype != np.uint64:
        a = a.astype(np.int64, copy=False).view(np.uint64) if a.dtype.kind in "iub" else a.astype(np.uint64)
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64).copy()).to(device())


def download_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").contiguous().numpy().view(np.uint64)


def to_engine(obj, session):
    """Rebind reference-style handles to engine shares of ``session`` (an
    ``mpfix.session.PartySession``)."""
    from .sharing import AShare, BShare
    if isinstance(obj, (AShare, BShare)):
        e = obj._engine((session.party,))
        if session._eng.dry:          # dry run: shapes only, like the reference's zero shares
            if isinstance(e, ES.AShare):
                return ES.AShare(_meta(e.values), e.width, e.frac, e.parties)
            return ES.BShare(_meta(e.words), e.m, e.axis, e.parties)
        return e
    if isinstance(obj, list):
        return [to_engine(v, session) for v in obj]
    if isinstance(obj, tuple):
        return tuple(to_engine(v, session) for v in obj)
    return obj


def _meta(t: torch.Tensor) -> torch.Tensor:
    return t if t.is_meta else torch.empty(t.shape, dtype=t.dtype, device="meta")


def from_engine(obj):
    from .sharing import AShare, BShare
    if isinstance(obj, ES.AShare):
        return AShare._from_engine(obj)
    if isinstance(obj, ES.BShare):
        return BShare._from_engine(obj)
    if isinstance(obj, list):
        return [from_engine(v) for v in obj]
    if isinstance(obj, tuple):
        return tuple(from_engine(v) for v in obj)
    return obj


def wrap_op(fn, name=None):
    """``op(session, *args, **kw)`` of the engine -> the reference signature
    over ``mpfix`` handles and sessions."""
    import functools

    @functools.wraps(fn)
    def op(session, *args, **kw):
        eng = session._eng
        a = [to_engine(v, session) for v in args]
        k = {key: to_engine(v, session) for key, v in kw.items()}
        return from_engine(fn(eng, *a, **k))
    if name:
        op.__name__ = name
    return op
