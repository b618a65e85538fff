"""``mpfix.session.PartySession`` (session.py:53-121) over the engine.

``PartySession(party, n_parties, mesh, store, rng=None, metrics=None)`` with
the reference's meaning: ``mesh`` is one party's fabric (an ``InProcHub``
mesh for party threads, ``NullMesh`` for dry runs, or ``None`` = NCCL over
the default ``torch.distributed`` group, one process per GPU); ``store`` is
a ``MaterialStore`` from ``memory_stores`` / ``device_store`` or a
``DemandCounter``. ``open_many`` returns numpy arrays (uint64 for arithmetic,
uint8 for bits) after one communication round, and records exactly the
reference's rounds and payload bytes.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import session as ESess
from ..metrics import CommMetrics
from . import transport
from ._bridge import device, download_u64, to_engine


class PartySession:
    def __init__(self, party: int, n_parties: int, mesh, store, rng: np.random.Generator | None = None,
                 metrics: CommMetrics | None = None):
        self.party = int(party)
        self.n_parties = int(n_parties)
        self.mesh = mesh
        self.store = store
        self.rng = rng if rng is not None else np.random.Generator(np.random.Philox(key=party))
        dry = bool(getattr(store, "dry", False))
        if dry and hasattr(store, "bind"):
            store.bind(self.party, self.n_parties)
        if isinstance(mesh, transport.NullMesh) or dry:
            comm = transport.NullComm(self.n_parties)
        elif isinstance(mesh, transport.InProcMesh):
            comm = mesh.comm
        else:
            comm = mesh
        dev = torch.device("meta") if dry else device()
        self._eng = ESess.PartySession(self.party, self.n_parties, comm, store, metrics=metrics, device=dev)
        self.metrics = self._eng.metrics

    def scope(self, name: str):
        return self.metrics.scope(name)

    def open_many(self, items: list) -> list[np.ndarray]:
        """One round; numpy results in item order (session.py:71-115)."""
        from .sharing import AShare, BShare
        for it in items:
            if not isinstance(it, (AShare, BShare)):
                raise TypeError(f"cannot open {type(it)}")
        opened = self._eng.open_many([to_engine(it, self) for it in items])
        out = []
        for it, t in zip(items, opened):
            if isinstance(it, AShare):
                out.append(np.zeros(it.shape, np.uint64) if t.is_meta else download_u64(t).reshape(it.shape))
            else:
                out.append(np.zeros(it.shape, np.uint8) if t.is_meta else t.cpu().numpy().reshape(it.shape))
        return out

    def open_arith(self, t) -> np.ndarray:
        return self.open_many([t])[0]

    def open_bits(self, b) -> np.ndarray:
        return self.open_many([b])[0]
