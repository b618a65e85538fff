"""Engine adapter for the B200 package (``paper_2402_02320_b200``), sim mode.

``dry(fn, n)`` runs a case against a DemandCounter with ``meta`` tensors (no
GPU needed): it exercises the whole protocol control flow, the material
demand and the op/communication ledger. ``run(fn, n)`` needs a GPU: dry run,
device dealer, live run, then exports every party's shares to numpy.
"""

from __future__ import annotations

import numpy as np
import torch

import paper_2402_02320_b200 as G
from paper_2402_02320_b200 import nn, nonlinear, protocols
from paper_2402_02320_b200.preprocessing import device_store
from paper_2402_02320_b200.session import SimSession, demands_by_name, dry_run

_M64 = (1 << 64) - 1


def _to_ring(v, width):
    a = np.asarray(v)
    if a.dtype != np.uint64:
        a = a.astype(np.int64).view(np.uint64)
    return a & np.uint64(_M64 if width == 64 else (1 << width) - 1)


def _bits_of(v, width):
    v = _to_ring(v, width)
    return ((v[..., None] >> np.arange(width, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)


def _encode(x, width, frac):
    s = np.floor(np.asarray(x, dtype=np.float64) * float(1 << frac))
    return _to_ring(s.astype(np.int64), width)


class GpuEngine:
    name = "b200"

    def __init__(self):
        for mod in (protocols, nonlinear, nn):
            for nm in dir(mod):
                if not nm.startswith("_"):
                    setattr(self, nm, getattr(mod, nm))
        self.bits_of, self.to_ring, self.encode = _bits_of, _to_ring, _encode
        self.EXP2_SQUARE = nonlinear.EXP2_SQUARE

    def params(self, **kw):
        return nonlinear.ApproxParams(**kw)

    def linear(self, w, b=None):
        return nn.LinearLayer(w, b)

    def deal_arith(self, s, values, width, frac=0, tag=0):
        return s.share_ring(_to_ring(values, width), width, frac, [1000 + tag, 2])

    def deal_fixed(self, s, floats, width, frac, tag=0):
        return self.deal_arith(s, _encode(floats, width, frac), width, frac, tag)

    def deal_bits(self, s, bits, tag=0):
        return s.share_bits(np.asarray(bits, np.uint8), [2000 + tag, 5])

    def dry(self, fn, n):
        counter = dry_run(lambda s: fn(self, s), n)
        return counter

    @staticmethod
    def export(v) -> np.ndarray:
        if isinstance(v, G.AShare):
            return v.values.cpu().numpy().view(np.uint64).copy()
        return v.bits.cpu().numpy().copy()

    def run(self, fn, n, seed=11, fuse=True):
        counter = dry_run(lambda s: fn(self, s), n)
        store = device_store(seed, n, counter.demands, needs_bits=counter.needs_bits)
        sess = SimSession(n, store)
        sess.fuse_ops = fuse
        out = fn(self, sess)
        torch.cuda.synchronize()
        res = {k: self.export(v) for k, v in out.items()}
        m = sess.metrics
        info = {"demands": demands_by_name(counter), "total": m.total.as_dict(),
                "ledger": {k: v.as_dict() for k, v in sorted(m.ledger.items())}}
        return res, info, sess


def run_party_threads(engine, fn, n, seed=11):
    """Party mode on one GPU: n threads, one PartySession (L=1) each, partial
    openings exchanged through a ThreadHub; returns per-party shares stacked
    on a leading party axis plus party 0's ledger."""
    import threading

    from paper_2402_02320_b200.session import PartySession, ThreadHub

    counter = dry_run(lambda s: fn(engine, s), n)
    hub = ThreadHub(n)
    hub.barrier = threading.Barrier(n, timeout=120)
    outs, errs, sessions = {}, {}, {}

    def worker(p):
        try:
            torch.cuda.set_device(0)
            store = device_store(seed, n, counter.demands, parties=(p,), needs_bits=counter.needs_bits)
            s = PartySession(p, n, hub.comm(p), store, device=torch.device("cuda", 0))
            sessions[p] = s
            outs[p] = fn(engine, s)
            torch.cuda.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs[p] = e
            hub.barrier.abort()

    ts = [threading.Thread(target=worker, args=(p,)) for p in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[min(errs)]
    res = {k: np.concatenate([GpuEngine.export(outs[p][k]) for p in range(n)]) for k in outs[0]}
    m = sessions[0].metrics
    info = {"demands": demands_by_name(counter), "total": m.total.as_dict(),
            "ledger": {k: v.as_dict() for k, v in sorted(m.ledger.items())}}
    return res, info, sessions
