"""Generate golden fixtures by running the REFERENCE itself (this container only).

    python tests/golden/make_golden.py            # all cases
    python tests/golden/make_golden.py mul_n2 ...  # a subset

For every case in ``tests/cases.py`` it imports ``mpfix`` from
``/root/reference/pkg/src`` (read-only; a throwaway matplotlib stub stands in
for the import in ``report.py:16-18``), runs the case with one thread per
party over the reference's own ``InProcHub`` with dealer seed 11 (as
``tests/helpers.py:17-49`` does), and stores every party's output shares, the
dry-run material demand and party 0's op ledger in ``tests/golden/<case>.npz``.
Also stores a Philox/dealer stream fixture (``dealer.npz``) straight from the
reference's ``generate_material``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from cases import CASES  # noqa: E402
from engines import ReferenceEngine  # noqa: E402


def save_case(eng, name):
    fn, n = CASES[name]
    out, info = eng.run(fn, n)
    arrays = {f"out__{k}": v for k, v in out.items()}
    arrays["info"] = np.frombuffer(json.dumps(info, sort_keys=True).encode(), dtype=np.uint8)
    arrays["n"] = np.asarray(n)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    return info


def save_dealer(eng):
    """Raw generate_material output for every kind, odd counts, n=3."""
    from mpfix.preprocessing import (bintriple_key, dabit_key, edabit_key, generate_material,
                                     mtriple_key, triple_key)
    keys = [triple_key(64), triple_key(32), mtriple_key(64, 3, 5, 2), bintriple_key(),
            dabit_key(64), dabit_key(32), edabit_key(64, 64), edabit_key(64, 23),
            edabit_key(32, 32), edabit_key(64, 40)]
    arrays = {}
    for key in keys:
        count = 13 if key.kind != 2 else 3
        per = generate_material(11, 3, key, count)
        for nm in per[0]:
            arrays[f"{key.name()}__{count}__{nm}"] = np.stack([per[p][nm] for p in range(3)])
    np.savez_compressed(os.path.join(HERE, "dealer.npz"), **arrays)


def save_dealer_files(eng):
    """Reference-written MPFXPRE1 files + manifest for the `reciprocal` and
    `batch_matmul` cases (seed 11): dry run on the reference, then
    preprocessing.dealer_generate / write_manifest (preprocessing.py:199-256)."""
    import shutil
    from mpfix.metrics import CommMetrics
    from mpfix.preprocessing import DemandCounter, dealer_generate, write_manifest
    from mpfix.session import PartySession
    from mpfix.transport import NullMesh
    for name in ("reciprocal", "batch_matmul"):
        fn, n = CASES[name]
        counter = DemandCounter(party=0)
        fn(eng, PartySession(0, n, NullMesh(0, n), counter, metrics=CommMetrics(0, n)))
        out = os.path.join(HERE, "files", name)
        shutil.rmtree(out, ignore_errors=True)
        dealer_generate(11, n, counter.demands, out)
        write_manifest(os.path.join(out, "manifest.json"), counter.demands)


def main(argv):
    eng = ReferenceEngine()
    names = argv or list(CASES)
    for nm in names:
        info = save_case(eng, nm)
        print(f"{nm}: rounds={info['total']['rounds']} demands={len(info['demands'])}")
    if not argv:
        save_dealer(eng)
        save_dealer_files(eng)
        print("dealer fixtures written")


if __name__ == "__main__":
    main(sys.argv[1:])
