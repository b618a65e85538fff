"""``mpfix.transport`` (transport.py:35-84, 239-259): the in-box fabrics.

* ``InProcHub(n).mesh(p)`` - party threads in one process, here on one GPU:
  each opening's partial is exchanged through a host rendezvous
  (``session.ThreadHub``) and reduced by a libmpx kernel.
* ``NullMesh(party, n)`` - dry runs: nothing is exchanged (the engine skips
  collectives when the store is a ``DemandCounter``).

One process per party per GPU needs no mesh object: pass ``mesh=None`` to
``PartySession`` and the openings are NCCL collectives over the default
``torch.distributed`` group. The TCP mesh (transport.py:87-236) is
cross-host transport, out of scope.
"""

from __future__ import annotations

from ..session import ThreadHub


class TransportError(RuntimeError):
    pass


class DesyncError(TransportError):
    pass


class HandshakeError(TransportError):
    pass


class InProcHub:
    def __init__(self, n_parties: int, timeout: float = 600.0):
        import threading
        self.n_parties = n_parties
        self._hub = ThreadHub(n_parties)
        self._hub.barrier = threading.Barrier(n_parties, timeout=timeout)

    def mesh(self, party: int) -> "InProcMesh":
        return InProcMesh(self, party)

    def abort(self) -> None:
        """Release every party blocked in an opening (a peer failed)."""
        self._hub.barrier.abort()


class InProcMesh:
    def __init__(self, hub: InProcHub, party: int):
        self.hub, self.party = hub, party
        self.comm = hub._hub.comm(party)

    def close(self) -> None:
        pass


class NullMesh:
    def __init__(self, party: int, n_parties: int):
        self.party, self.n_parties = party, n_parties

    def close(self) -> None:
        pass


class NullComm:
    """Communicator of a dry run: the session never calls it."""

    def __init__(self, n: int):
        self.world = n

    def allreduce_sum_(self, flat):
        raise TransportError("NullMesh cannot open live shares (dry runs only)")

    def allgather(self, flat):
        raise TransportError("NullMesh cannot open live shares (dry runs only)")
