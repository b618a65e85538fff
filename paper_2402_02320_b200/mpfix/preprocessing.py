"""``mpfix.preprocessing`` (preprocessing.py:61-403) over the device dealer.

Same key names, demand accounting and store semantics as the reference; the
material is dealt on the GPU by the engine's Philox dealer (bit-exact with
``generate_material``) and stays in HBM. ``memory_stores`` returns one store
per party, ``DemandCounter(party)`` sizes a dry run, ``FileStore`` reads the
reference's ``MPFXPRE1`` files, ``generate_material`` / ``dealer_generate``
produce the reference's arrays and files from the device dealer.
"""

from __future__ import annotations

from .. import material_io as MIO
from .. import preprocessing as EP
from ..preprocessing import (MaterialKey, MaterialStore, PreprocessingExhausted, bintriple_key, dabit_key,
                             edabit_key, mtriple_key, triple_key)
from ._bridge import device


class DemandCounter(EP.DemandCounter):
    """Dry-run store for one party (preprocessing.py:369-403)."""

    def __init__(self, party: int = 0):
        super().__init__((party,), 0)
        self.party = party

    def bind(self, party: int, n_parties: int) -> None:
        self.parties, self.party, self.n_parties = (party,), party, n_parties


def memory_stores(seed: int, n_parties: int, demands: dict) -> list[MaterialStore]:
    """Dealer output kept on the device, one store per party (preprocessing.py:356-366)."""
    dev = device()
    return [EP.device_store(seed, n_parties, demands, parties=(p,), device=dev) for p in range(n_parties)]


class FileStore(MIO.FileStore):
    """Store backed by the per-party directory the dealer wrote (preprocessing.py:335-353)."""

    def __init__(self, root_dir: str, party: int, n_parties: int | None = None):
        import os
        if n_parties is None:
            n_parties = _n_from_files(os.path.join(root_dir, f"party{party}"))
        super().__init__(root_dir, (party,), n_parties, device())
        self.party = party


def _n_from_files(party_dir: str) -> int:
    import os
    if not os.path.isdir(party_dir):
        raise FileNotFoundError(f"no preprocessing directory {party_dir}")
    for nm in sorted(os.listdir(party_dir)):
        if nm.endswith(".bin"):
            return MIO.read_material_file(os.path.join(party_dir, nm))[2]
    return 0


def generate_material(seed: int, n_parties: int, key: MaterialKey, count: int) -> list[dict]:
    """Per-party arrays in the reference layout (preprocessing.py:128-174), dealt on the GPU."""
    dealer = EP.Dealer(seed, n_parties, 0, n_parties, device())
    arrays = dealer.generate(key, count, need_bits=True)
    return [MIO.export_arrays(key, count, arrays, p) for p in range(n_parties)]


def dealer_generate(seed: int, n_parties: int, demands: dict, out_dir: str) -> None:
    MIO.dealer_generate(seed, n_parties, demands, out_dir, device=device())


write_material_file = MIO.write_material_file
read_material_file = MIO.read_material_file
write_manifest = MIO.write_manifest
read_manifest = MIO.read_manifest

__all__ = ["MaterialKey", "MaterialStore", "PreprocessingExhausted", "DemandCounter", "FileStore",
           "memory_stores", "generate_material", "dealer_generate", "triple_key", "mtriple_key",
           "bintriple_key", "dabit_key", "edabit_key", "write_material_file", "read_material_file",
           "write_manifest", "read_manifest"]
