"""Engine adapters: one namespace per implementation for ``tests/cases.py``.

* ``ReferenceEngine`` imports the reference package from ``/root/reference``
  (golden-fixture generation only; it never runs on the GPU box).
* ``OracleEngine`` drives the CPU oracle (``oracle/``).
* ``GpuEngine`` (in ``tests/gpu_engine.py``) drives the B200 package.

``run(fn, n, seed)`` returns ``(outputs, info)`` where ``outputs`` maps each
returned name to a numpy array with a leading party axis (uint64 arithmetic
shares, uint8 bits) and ``info`` holds the material demand and party 0's
operation ledger.
"""

from __future__ import annotations

import os
import sys
import tempfile
import threading
import types

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

REFERENCE_SRC = "/root/reference/pkg/src"
REFERENCE_TESTS = "/root/reference/pkg/tests"


# ---------------------------------------------------------------------------
# CPU oracle


class OracleEngine:
    name = "oracle"

    def __init__(self):
        import oracle as O
        self.O = O
        for nm in ("mul", "batch_matmul", "and_gate", "bit2a", "compose", "decompose",
                   "binary_add", "public_add_bits", "gt", "const_share", "add_const",
                   "truncate", "unsigned_truncate", "scale_fixed", "evaluate_poly",
                   "evaluate_square_completed", "lmo", "max_vec", "reciprocal",
                   "exponentiation", "logarithm", "baseline_exp", "attention_exp", "relu",
                   "maxcut", "softmax", "softmax_parts", "attention_block", "linear_layer",
                   "mlp_forward", "bits_of", "to_ring", "encode", "EXP2_SQUARE"):
            setattr(self, nm, getattr(O, nm))

    def params(self, **kw):
        return self.O.Params(**kw)

    def linear(self, w, b=None):
        return self.O.Linear(w, b)

    def deal_arith(self, s, values, width, frac=0, tag=0):
        return self.O.AShare(self.O.deal_inputs_arith(values, s.n, width, [1000 + tag, 2]), width, frac)

    def deal_fixed(self, s, floats, width, frac, tag=0):
        return self.deal_arith(s, self.O.encode(np.asarray(floats, np.float64), width, frac), width,
                               frac, tag)

    def deal_bits(self, s, bits, tag=0):
        return self.O.BShare(self.O.deal_inputs_bits(bits, s.n, [2000 + tag, 5]))

    def run(self, fn, n, seed=11):
        out, sess = self.O.simulate(lambda s: fn(self, s), n, seed)
        res = {}
        for k, v in out.items():
            res[k] = v.values.copy() if isinstance(v, self.O.AShare) else v.bits.copy()
        info = {"demands": dict(sorted(sess.store._count.items())),
                "total": sess.ledger.total.as_dict(),
                "ledger": {k: v.as_dict() for k, v in sorted(sess.ledger.by_scope.items())}}
        return res, info


# ---------------------------------------------------------------------------
# The reference itself (golden generation only)


def _matplotlib_stub() -> str:
    d = tempfile.mkdtemp(prefix="mplstub_")
    os.makedirs(os.path.join(d, "matplotlib"))
    with open(os.path.join(d, "matplotlib", "__init__.py"), "w") as fh:
        fh.write("def use(*a, **k):\n    pass\n")
    with open(os.path.join(d, "matplotlib", "pyplot.py"), "w") as fh:
        fh.write("def __getattr__(n):\n    return lambda *a, **k: None\n")
    return d


class ReferenceEngine:
    name = "reference"

    def __init__(self):
        for p in (REFERENCE_SRC, REFERENCE_TESTS, _matplotlib_stub()):
            if p not in sys.path:
                sys.path.insert(0, p)
        import mpfix
        from mpfix import nn, nonlinear, protocols, ring
        import helpers  # reference tests/helpers.py
        self.mpfix, self.helpers, self.ring = mpfix, helpers, ring
        for mod in (protocols, nonlinear, nn):
            for nm in dir(mod):
                if not nm.startswith("_"):
                    setattr(self, nm, getattr(mod, nm))
        self.bits_of, self.to_ring, self.encode = ring.bits_of, ring.to_ring, ring.encode
        self.EXP2_SQUARE = nonlinear.EXP2_SQUARE

    def params(self, **kw):
        return self.mpfix.nonlinear.ApproxParams(**kw)

    def linear(self, w, b=None):
        return self.mpfix.nn.LinearLayer(w, b)

    def deal_arith(self, s, values, width, frac=0, tag=0):
        return self.helpers.deal_arith(s, values, width, frac, tag=tag)

    def deal_fixed(self, s, floats, width, frac, tag=0):
        return self.helpers.deal_fixed(s, floats, width, frac, tag=tag)[0]

    def deal_bits(self, s, bits, tag=0):
        return self.helpers.deal_bits(s, bits, tag=tag)

    def run(self, fn, n, seed=11):
        from mpfix.metrics import CommMetrics
        from mpfix.preprocessing import DemandCounter, memory_stores
        from mpfix.session import PartySession
        from mpfix.sharing import AShare
        from mpfix.transport import InProcHub, NullMesh

        counter = DemandCounter(party=0)
        fn(self, PartySession(0, n, NullMesh(0, n), counter, metrics=CommMetrics(0, n)))
        stores = memory_stores(seed, n, dict(counter.demands))
        hub = InProcHub(n)
        outs, errs, sessions = {}, {}, {}

        def worker(p):
            try:
                s = PartySession(p, n, hub.mesh(p), stores[p], metrics=CommMetrics(p, n))
                sessions[p] = s
                outs[p] = fn(self, s)
            except BaseException as e:  # noqa: BLE001
                errs[p] = e

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
