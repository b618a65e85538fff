"""Engine adapter for the reference-compatible facade (``paper_2402_02320_b200.mpfix``).

Mirrors ``engines.ReferenceEngine`` line for line, but every import resolves
to the facade: reference-style callers (one ``PartySession`` per party thread
over ``InProcHub`` meshes, numpy ``AShare`` / ``BShare`` handles, the
``tests/helpers.py`` dealing functions) drive the B200 engine unmodified.
"""

from __future__ import annotations

import threading

import numpy as np

import mpfix_helpers as H


class FacadeEngine:
    name = "facade"

    def __init__(self):
        from paper_2402_02320_b200 import mpfix
        from paper_2402_02320_b200.mpfix import nn, nonlinear, protocols, ring
        self.mpfix, self.ring = mpfix, ring
        for mod in (protocols, nonlinear, nn):
            for nm in dir(mod):
                if not nm.startswith("_"):
                    setattr(self, nm, getattr(mod, nm))
        self.bits_of, self.to_ring, self.encode = ring.bits_of, ring.to_ring, ring.encode
        from paper_2402_02320_b200.nonlinear import EXP2_SQUARE
        self.EXP2_SQUARE = EXP2_SQUARE

    def params(self, **kw):
        return self.mpfix.nonlinear.ApproxParams(**kw)

    def linear(self, w, b=None):
        return self.mpfix.nn.LinearLayer(w, b)

    def deal_arith(self, s, values, width, frac=0, tag=0):
        return H.deal_arith(s, values, width, frac, tag=tag)

    def deal_fixed(self, s, floats, width, frac, tag=0):
        return H.deal_fixed(s, floats, width, frac, tag=tag)[0]

    def deal_bits(self, s, bits, tag=0):
        return H.deal_bits(s, bits, tag=tag)

    def run(self, fn, n, seed=11):
        import torch
        from paper_2402_02320_b200.mpfix.metrics import CommMetrics
        from paper_2402_02320_b200.mpfix.preprocessing import DemandCounter, memory_stores
        from paper_2402_02320_b200.mpfix.session import PartySession
        from paper_2402_02320_b200.mpfix.sharing import AShare
        from paper_2402_02320_b200.mpfix.transport import InProcHub, NullMesh

        counter = DemandCounter(party=0)
        fn(self, PartySession(0, n, NullMesh(0, n), counter, metrics=CommMetrics(0, n)))
        stores = memory_stores(seed, n, dict(counter.demands))
        hub = InProcHub(n, timeout=300)
        outs, errs, sessions = {}, {}, {}

        def worker(p):
            try:
                torch.cuda.set_device(0)
                s = PartySession(p, n, hub.mesh(p), stores[p], metrics=CommMetrics(p, n))
                sessions[p] = s
                outs[p] = fn(self, s)
            except BaseException as e:  # noqa: BLE001
                errs[p] = e
                hub.abort()

        ts = [threading.Thread(target=worker, args=(p,)) for p in range(n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[min(errs)]
        res = {}
        for k in outs[0]:
            per = [outs[p][k] for p in range(n)]
            res[k] = np.stack([v.values if isinstance(v, AShare) else v.bits for v in per])
        m = sessions[0].metrics
        info = {"demands": {key.name(): c for key, c in sorted(counter.demands.items(),
                                                               key=lambda kv: kv[0].name()) if c > 0},
                "total": m.total.as_dict(),
                "ledger": {k: v.as_dict() for k, v in sorted(m.ledger.items())}}
        return res, info
