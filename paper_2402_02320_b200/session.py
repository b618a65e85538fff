"""Party sessions: where every opening happens (reference: session.py:53-121).

Two deployments share one protocol code path:

* ``SimSession`` - all n parties on one GPU (the reference's ``run_all`` with
  ``InProcHub``): shares carry all n parties on the leading axis and an
  opening is the local reduction the mask kernel already performed, so the
  sim-mode protocols use fused single-pass kernels.
* ``PartySession`` - one process per party per GPU (``torchrun``), the
  reference's TCP/in-proc mesh replaced by NCCL over NVLink: arithmetic
  openings are one ``all_reduce(SUM)`` on int64 words (two's-complement wrap
  = Z_2^64, bit-exact in any reduction order); binary openings are an
  ``all_gather`` of packed words folded with an XOR kernel (NCCL has no XOR).

Either way the ledger records the reference's logical payload: (n-1) x the
opened bytes per round (u4 for w<=32, u8 otherwise, bits packed 8/byte).

A session whose store is a ``DemandCounter`` is a dry run (NullMesh +
DemandCounter in the reference, runner.py:49-58): tensors are ``meta``, no
kernel launches and no collectives happen, but the demand and ledger are
recorded exactly.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import kernels as K
from .metrics import CommMetrics
from .preprocessing import DemandCounter, MaterialKey, device_store
from .ring import decode
from .sharing import AShare, BShare


def arith_payload(width: int, count: int) -> int:
    """Per-peer bytes of an opened arithmetic tensor (session.py:24-29,47-50)."""
    return count * (4 if width <= 32 else 8)


def bits_payload(count: int) -> int:
    return (count + 7) // 8


class _Session:
    world = 1

    def __init__(self, parties, n_parties, store, metrics, device):
        self.parties = tuple(parties)
        self.n_parties = int(n_parties)
        self.store = store
        self.dry = bool(getattr(store, "dry", False))
        self.device = torch.device("meta") if self.dry else torch.device(device)
        me = self.parties[0] if len(self.parties) == 1 else 0
        self.metrics = metrics if metrics is not None else CommMetrics(me, self.n_parties)
        self._peers = [p for p in range(self.n_parties) if p != me]
        self._step = 0

    # -- layout ------------------------------------------------------------------
    @property
    def L(self) -> int:
        return len(self.parties)

    @property
    def p0(self) -> int:
        return self.parties.index(0) if 0 in self.parties else -1

    @property
    def fused(self) -> bool:
        """All parties local and live: an opening needs no communication."""
        return self.world == 1 and not self.dry and self.L == self.n_parties

    def alloc(self, shape) -> torch.Tensor:
        return torch.empty(tuple(shape), dtype=torch.int64, device=self.device)

    def scope(self, name: str):
        return self.metrics.scope(name)

    # -- rounds ------------------------------------------------------------------
    def _account(self, payload_bytes: int) -> None:
        self._step += 1
        for peer in self._peers:
            self.metrics.record_send(peer, payload_bytes)
        self.metrics.record_round()

    def exchange(self, arith=(), bits=(), payload: int | None = None):
        """One communication round over partial openings.

        ``arith``: list of (partial sums int64[n], width); ``bits``: list of
        partial XOR words. Returns the opened tensors (arith first, then bits).
        ``payload`` overrides the logical per-peer byte count when the kernel
        layout differs from the reference's item list (carry levels).
        """
        if payload is None:
            payload = sum(arith_payload(w, t.numel()) for t, w in arith) + \
                sum(bits_payload(t.numel()) for t in bits)
        self._account(payload)
        outs = [t for t, _ in arith] + list(bits)
        if self.world == 1 and not self.dry and self.L != self.n_parties:
            raise RuntimeError(f"parties {self.parties} of {self.n_parties} hold partial shares but the session "
                               "has no communicator: pass a mesh or init torch.distributed")
        if self.world > 1 and not self.dry:
            outs = self._collective([t for t, _ in arith], list(bits))
        return outs

    def _collective(self, arith, bits):  # pragma: no cover - party mode only
        raise NotImplementedError

    # -- public API (session.py:71-121) ------------------------------------------
    def open_many(self, items: list) -> list[torch.Tensor]:
        """Open several shared tensors in one round. Returns device tensors:
        int64 ring words (masked) for AShare, uint8 bits for BShare."""
        arith, bits, order = [], [], []
        for it in items:
            if isinstance(it, AShare):
                t = self.alloc((it.size,))
                K.open_sum(t, it.values, it.L, it.size, it.width)
                arith.append((t, it.width))
                order.append(("a", it))
            elif isinstance(it, BShare):
                t = self.alloc((it.rows,))
                K.open_xor(t, it.words, it.L, it.rows)
                bits.append(t)
                order.append(("b", it))
            else:
                raise TypeError(f"cannot open {type(it)}")
        payload = sum(arith_payload(w, t.numel()) for t, w in arith) + \
            sum(bits_payload(it.size) for k, it in order if k == "b")
        opened = self.exchange(arith, bits, payload=payload)
        na = len(arith)
        res, ia, ib = [], 0, 0
        for kind, it in order:
            if kind == "a":
                t = opened[ia]
                ia += 1
                if self.world > 1 and not self.dry and it.width < 64:
                    K.ring_lin(t, t, 1, None, 0, 0, None, 1, t.numel(), it.width, -1)
                res.append(t.view(it.shape))
            else:
                w = opened[na + ib]
                ib += 1
                if it.axis:
                    out = torch.empty((it.rows, it.m), dtype=torch.uint8, device=self.device)
                    K.bits_unpack(out, w, it.rows, it.m)
                    res.append(out.view(it.shape))
                else:
                    res.append(w.to(torch.uint8).view(it.shape))
        return res

    def open_arith(self, t: AShare) -> torch.Tensor:
        return self.open_many([t])[0]

    def open_bits(self, b: BShare) -> torch.Tensor:
        return self.open_many([b])[0]

    def open_fixed(self, t: AShare) -> np.ndarray:
        """Open and decode to float64 on the host (harness helper)."""
        v = self.open_arith(t)
        return decode(v, t.width, t.frac).cpu().numpy()

    # -- input sharing (scenarios.py:54-84, tests/helpers.py:52-78) ----------------
    def share_ring(self, enc, width: int, frac: int, key) -> AShare:
        """Deterministic additive sharing of a public ring tensor: parties
        1..n-1 draw Philox(key) elements in order, party 0 holds the difference."""
        enc_t = _as_words(enc, self.device)
        n = enc_t.numel()
        vals = self.alloc((self.L,) + tuple(enc_t.shape))
        kk = _philox_key(key)
        if not self.dry:
            draws = {}
            for p in range(1, self.n_parties):
                if p in self.parties or 0 in self.parties:
                    d = torch.empty(n, dtype=torch.int64, device=self.device)
                    K.philox_elems(d, kk, (p - 1) * 2 * max(n, 1), n, width)
                    draws[p] = d
            for li, p in enumerate(self.parties):
                dst = vals[li].view(-1)
                if p == 0:
                    acc = enc_t.reshape(-1).clone()
                    for q in range(1, self.n_parties):
                        K.ring_lin(acc, acc, 1, draws[q], (1 << 64) - 1, 0, None, 1, n, width, -1)
                    K.ring_lin(dst, acc, 1, None, 0, 0, None, 1, n, width, -1)
                else:
                    dst.copy_(draws[p])
        return AShare(vals, width, frac, self.parties)

    def share_fixed(self, floats, width: int, frac: int, key) -> AShare:
        from .ring import encode
        return self.share_ring(encode(floats, width, frac, self.device), width, frac, key)

    def share_bits(self, bits, key) -> BShare:
        """XOR analogue of ``share_ring`` (one Philox byte per bit)."""
        arr = np.asarray(bits.cpu().numpy() if isinstance(bits, torch.Tensor) else bits, dtype=np.uint8)
        shape = arr.shape
        n = arr.size
        kk = _philox_key(key)
        flat_w = (n + 63) // 64 + 2
        packed = np.zeros(flat_w * 64, dtype=np.uint8)
        packed[:n] = arr.reshape(-1) & 1
        secret = np.packbits(packed, bitorder="little").view(np.uint64).view(np.int64)
        axis = len(shape) >= 1 and shape[-1] <= 64
        m = shape[-1] if axis else 1
        rows_shape = shape[:-1] if axis else shape
        rows = math.prod(rows_shape)
        words = self.alloc((self.L,) + tuple(rows_shape))
        if not self.dry:
            sec = torch.from_numpy(secret.copy()).to(self.device)
            draw_u32 = (max(n, 1) + 3) // 4
            flats = {}
            for p in range(1, self.n_parties):
                if p in self.parties or 0 in self.parties:
                    f = torch.zeros(flat_w, dtype=torch.int64, device=self.device)
                    K.philox_bits(f, kk, (p - 1) * draw_u32, n)
                    flats[p] = f
            for li, p in enumerate(self.parties):
                if p == 0:
                    acc = sec.clone()
                    for q in range(1, self.n_parties):
                        K.bits_op(acc, acc, flats[q], 0, 1, flat_w, 64)
                    src = acc
                else:
                    src = flats[p]
                K.bits_flat_to_rows(words[li].view(-1), src.data_ptr(), 0, rows, m)
        return BShare(words, m, axis, self.parties)


def _as_words(enc, device) -> torch.Tensor:
    if isinstance(enc, torch.Tensor):
        t = enc.to(torch.int64) if enc.dtype != torch.uint64 else enc.view(torch.int64)
        return t.to(device) if t.device != device else t
    a = np.asarray(enc)
    if a.dtype != np.uint64:
        a = a.astype(np.int64).view(np.uint64)
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy())
    if device.type == "meta":
        return torch.empty(t.shape, dtype=torch.int64, device="meta")
    return t.to(device)


def _philox_key(key) -> tuple[int, int]:
    if isinstance(key, (int, np.integer)):
        k = int(key)
        return (k & ((1 << 64) - 1), k >> 64)
    words = [int(v) for v in np.asarray(key, dtype=np.uint64).ravel()] + [0, 0]
    return (words[0], words[1])


class SimSession(_Session):
    """All n parties on one GPU; opening = local reduction over the party axis."""

    def __init__(self, n_parties: int, store, metrics: CommMetrics | None = None, device="cuda"):
        super().__init__(range(n_parties), n_parties, store, metrics, device)
        self.party = None


class DistComm:
    """Collectives over a torch.distributed group: NCCL over NVLink on B200
    (gloo on CPU for host-logic tests). Communication only - no arithmetic."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce_sum_(self, flat: torch.Tensor) -> None:
        """In-place int64 sum over ranks; two's-complement wrap = Z_2^64."""
        self.dist.all_reduce(flat, op=self.dist.ReduceOp.SUM, group=self.group)

    def allgather(self, flat: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.world, flat.numel()), dtype=flat.dtype, device=flat.device)
        if flat.is_cuda:
            self.dist.all_gather_into_tensor(out, flat, group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), flat, group=self.group)
        return out


class ThreadHub:
    """Test harness: n party threads on ONE GPU exchanging partial openings by
    host rendezvous (no device-side waiting). Emulates the NCCL party layer so
    the per-round mask -> exchange -> finish path runs bit-exactly on 1 GPU."""

    def __init__(self, n: int):
        import threading
        self.n = n
        self.barrier = threading.Barrier(n)
        self.slots = [None] * n

    def comm(self, rank: int) -> "ThreadComm":
        return ThreadComm(self, rank)


class ThreadComm:
    def __init__(self, hub: ThreadHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.n

    def allgather(self, flat: torch.Tensor) -> torch.Tensor:
        torch.cuda.current_stream().synchronize()
        self.hub.slots[self.rank] = flat
        self.hub.barrier.wait()
        out = torch.stack(self.hub.slots)
        torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()
        return out

    def allreduce_sum_(self, flat: torch.Tensor) -> None:
        g = self.allgather(flat)
        K.open_sum(flat, g, self.world, flat.numel(), 64)


class LoopbackComm:
    """Timing stand-in for ONE party of an n-party deployment on one GPU: the
    collectives keep (sum) or replicate (gather) this party's own partial, so
    opened values are meaningless, but every kernel, tensor size and round
    of the one-party-per-GPU (L = 1) path runs exactly as deployed; it is
    CUDA-graph capturable. bench.py reports the party's compute time per step
    with it (the communication is what the n-GPU run adds)."""

    def __init__(self, n: int):
        self.world = n

    def allreduce_sum_(self, flat: torch.Tensor) -> None:
        return None

    def allgather(self, flat: torch.Tensor) -> torch.Tensor:
        return flat.unsqueeze(0).expand(self.world, flat.numel()).contiguous()


class PartySession(_Session):
    """One party per process/GPU; openings are collectives over the party group.

    Signature mirrors the reference's ``PartySession(party, n_parties, mesh,
    store, rng, metrics)`` (session.py:53-64). ``mesh`` is the communicator:
    None = the default torch.distributed group over NCCL (``DistComm``), or
    any object with ``world``, ``allreduce_sum_`` and ``allgather``.
    """

    def __init__(self, party: int, n_parties: int, mesh=None, store=None, rng=None,
                 metrics: CommMetrics | None = None, device=None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                else torch.device("cpu")
        super().__init__((party,), n_parties, store, metrics, device)
        self.party = party
        if mesh is None:
            import torch.distributed as dist
            mesh = DistComm() if dist.is_available() and dist.is_initialized() else None
        self.comm = mesh
        self.world = mesh.world if mesh is not None else 1
        if self.world not in (1, n_parties):
            raise ValueError("one rank per party expected")
        if mesh is None and n_parties > 1 and store is not None and not self.dry:
            raise RuntimeError(f"party {party} of {n_parties}: no communicator (mesh=None and torch.distributed "
                               "is not initialised); openings would silently use the local share only")

    def _collective(self, arith, bits):
        outs = []
        if arith:
            cover = _covering(arith)
            if cover is not None:          # the round's payloads tile one buffer: reduce it in place
                self.comm.allreduce_sum_(cover)
                self.metrics.physical_bytes += cover.numel() * 8
                outs.extend(arith)
            else:
                flat = torch.cat([t.reshape(-1) for t in arith])
                self.comm.allreduce_sum_(flat)
                self.metrics.physical_bytes += flat.numel() * 8
                off = 0
                for t in arith:
                    outs.append(flat[off:off + t.numel()].view(t.shape))
                    off += t.numel()
        if bits:
            cover = _covering(bits)
            flat = cover if cover is not None else torch.cat([t.reshape(-1) for t in bits])
            gathered = self.comm.allgather(flat)
            self.metrics.physical_bytes += flat.numel() * 8 * (self.world - 1)
            K.open_xor(flat, gathered, self.world, flat.numel())   # XOR of every party's partial, in place
            if cover is not None:
                outs.extend(bits)
            else:
                off = 0
                for t in bits:
                    outs.append(flat[off:off + t.numel()].view(t.shape))
                    off += t.numel()
        return outs


def _covering(ts):
    """A flat contiguous view covering exactly the tensors ``ts`` when they
    tile one range of one storage (any order), else None."""
    if len(ts) == 1:
        t = ts[0]
        return t.view(-1) if t.is_contiguous() else None
    if any(not t.is_contiguous() or t.untyped_storage().data_ptr() != ts[0].untyped_storage().data_ptr()
           for t in ts):
        return None
    spans = sorted((t.data_ptr(), t.numel()) for t in ts)
    for (p, n), (q, _) in zip(spans, spans[1:]):
        if p + 8 * n != q:
            return None
    base = ts[0].untyped_storage()
    lo = spans[0][0]
    total = sum(n for _, n in spans)
    off = (lo - base.data_ptr()) // 8
    return torch.empty(0, dtype=torch.int64, device=ts[0].device).set_(base, off, (total,), (1,))


# ---------------------------------------------------------------------------
# Harness: dry run -> device dealer -> live run (tests/helpers.py:17-49)


def dry_run(fn, n_parties: int, parties=None):
    parties = tuple(range(n_parties)) if parties is None else tuple(parties)
    counter = DemandCounter(parties, n_parties)
    sess = SimSession(n_parties, counter) if len(parties) == n_parties else None
    if sess is None:
        raise ValueError("dry_run builds sim sessions; use PartySession with a DemandCounter")
    fn(sess)
    return counter


def run_sim(fn, n_parties: int, seed: int = 11, device="cuda"):
    """Run ``fn(session)`` once for all parties on one GPU. Returns (result, session)."""
    counter = dry_run(fn, n_parties)
    store = device_store(seed, n_parties, counter.demands, device=device, needs_bits=counter.needs_bits)
    sess = SimSession(n_parties, store, device=device)
    return fn(sess), sess


def demands_by_name(counter: DemandCounter) -> dict[str, int]:
    return {k.name(): c for k, c in sorted(counter.demands.items(), key=lambda kv: kv[0].name()) if c > 0}


__all__ = ["SimSession", "PartySession", "DistComm", "ThreadHub", "LoopbackComm", "run_sim", "dry_run",
           "demands_by_name", "MaterialKey"]
