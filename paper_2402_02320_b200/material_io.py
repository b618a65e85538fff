"""Dealer material files: the reference's ``MPFXPRE1`` format on the B200 store.

Byte-compatible with ``preprocessing.py:181-256`` of the reference: one file
per party per material key, header ``<8sHBBHHQ4I`` (magic, version, kind,
width, party, n_parties, count, 4 params), then the kind's payload blocks in
file order (arithmetic parts as little-endian u64, bit parts one byte per
bit), plus a JSON manifest of counts. Files written by the reference's
``dealer_generate`` load into ``FileStore`` and drive the GPU protocols
bit-exactly; ``dealer_generate`` here writes byte-identical files from the
on-device dealer.

Device <-> file layout conversion (flat packed bit streams <-> one byte per
bit) runs in libmpx kernels (``mpx_bits_pack`` / ``mpx_bits_unpack``).
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import torch

from . import kernels as K
from .preprocessing import (KIND_BIN_TRIPLE, KIND_DABIT, KIND_EDABIT, KIND_MATRIX_TRIPLE, KIND_TRIPLE,
                            Dealer, MaterialKey, MaterialStore, PreprocessingExhausted, _words)

MAGIC = b"MPFXPRE1"
VERSION = 1
HEADER = struct.Struct("<8sHBBHHQ4I")


def payload_blocks(key: MaterialKey, count: int) -> list[tuple[str, str, tuple]]:
    """(array name, dtype, shape) in file order (preprocessing.py:181-196)."""
    if key.kind == KIND_TRIPLE:
        return [(n, "<u8", (count,)) for n in ("a", "b", "c")]
    if key.kind == KIND_MATRIX_TRIPLE:
        m, k, r = key.params
        return [("a", "<u8", (count, m, k)), ("b", "<u8", (count, k, r)), ("c", "<u8", (count, m, r))]
    if key.kind == KIND_BIN_TRIPLE:
        return [(n, "u1", (count,)) for n in ("a", "b", "c")]
    if key.kind == KIND_DABIT:
        return [("arith", "<u8", (count,)), ("bit", "u1", (count,))]
    if key.kind == KIND_EDABIT:
        return [("arith", "<u8", (count,)), ("bits", "u1", (count, key.params[0]))]
    raise ValueError(f"unknown material kind {key.kind}")


def write_material_file(path: str, key: MaterialKey, party: int, n_parties: int, count: int,
                        arrays: dict) -> None:
    """Host arrays in the reference layout -> one party file (preprocessing.py:199-210)."""
    params = list(key.params) + [0] * (4 - len(key.params))
    with open(path, "wb") as fh:
        fh.write(HEADER.pack(MAGIC, VERSION, key.kind, key.width, party, n_parties, count, *params))
        for name, dtype, shape in payload_blocks(key, count):
            arr = np.ascontiguousarray(arrays[name], dtype=dtype)
            if arr.shape != shape:
                raise ValueError(f"{name}: expected shape {shape}, got {arr.shape}")
            fh.write(arr.tobytes())


def read_material_file(path: str):
    """-> (key, party, n_parties, count, arrays in the reference layout) (preprocessing.py:213-229)."""
    with open(path, "rb") as fh:
        raw = fh.read(HEADER.size)
        magic, version, kind, width, party, n_parties, count, p0, p1, p2, p3 = HEADER.unpack(raw)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a preprocessing file")
        if version != VERSION:
            raise ValueError(f"{path}: unsupported version {version}")
        nparams = {KIND_EDABIT: 1, KIND_MATRIX_TRIPLE: 3}.get(kind, 0)
        key = MaterialKey(kind, width, tuple((p0, p1, p2, p3))[:nparams])
        arrays = {}
        for name, dtype, shape in payload_blocks(key, count):
            n_items = int(np.prod(shape)) if shape else 0
            buf = fh.read(n_items * np.dtype(dtype).itemsize)
            if len(buf) != n_items * np.dtype(dtype).itemsize:
                raise ValueError(f"{path}: truncated payload")
            arrays[name] = np.frombuffer(buf, dtype=dtype).reshape(shape).copy()
    return key, party, n_parties, count, arrays


def write_manifest(path: str, demands: dict) -> None:
    named = {(k.name() if isinstance(k, MaterialKey) else k): int(c) for k, c in demands.items()}
    with open(path, "w") as fh:
        json.dump(named, fh, indent=2, sort_keys=True)
        fh.write("\n")


def read_manifest(path: str) -> dict[MaterialKey, int]:
    with open(path) as fh:
        return {MaterialKey.from_name(n): int(c) for n, c in json.load(fh).items()}


# ---------------------------------------------------------------------------
# device layout <-> reference layout


def _unpack_bits(words: torch.Tensor, count: int) -> np.ndarray:
    """Flat packed stream int64[nw] -> uint8[count], one byte per bit."""
    nw = (count + 63) // 64
    out = torch.empty(nw * 64, dtype=torch.uint8, device=words.device)
    if nw:
        K.bits_unpack(out, words[:nw].contiguous(), nw, 64)
    return out[:count].cpu().numpy()


def _pack_bits(bits: np.ndarray, device) -> torch.Tensor:
    """uint8[count] (one byte per bit) -> flat packed int64[ceil(count/64)+2]."""
    count = bits.size
    nw = (count + 63) // 64
    padded = np.zeros(nw * 64, dtype=np.uint8)
    padded[:count] = bits.reshape(-1) & 1
    out = torch.zeros(_words(count), dtype=torch.int64, device=device)
    if nw:
        K.bits_pack(out, torch.from_numpy(padded).to(device), nw, 64)
    return out


def export_arrays(key: MaterialKey, count: int, dev_arrays: dict, li: int) -> dict:
    """Local party ``li`` of device material -> reference-layout numpy arrays."""
    out = {}
    for name, dtype, shape in payload_blocks(key, count):
        t = dev_arrays[name][li]
        if dtype == "u1":
            out[name] = _unpack_bits(t, int(np.prod(shape))).reshape(shape)
        else:
            out[name] = t.reshape(shape).cpu().numpy().view(np.uint64)
    return out


def import_arrays(key: MaterialKey, count: int, per_party: list[dict], device) -> dict:
    """Reference-layout arrays of the local parties -> device store layout."""
    dev = {}
    for name, dtype, shape in payload_blocks(key, count):
        if dtype == "u1":
            dev[name] = torch.stack([_pack_bits(a[name], device) for a in per_party])
        else:
            dev[name] = torch.stack([torch.from_numpy(np.ascontiguousarray(a[name]).view(np.int64)).to(device)
                                     for a in per_party]).reshape((len(per_party),) + shape)
    return dev


# ---------------------------------------------------------------------------
# stores and the file-writing dealer


class FileStore(MaterialStore):
    """Store backed by dealer files on disk (preprocessing.py:335-353); loads a
    key's files for the local parties on first use."""

    def __init__(self, root_dir: str, parties, n_parties: int, device="cuda"):
        super().__init__(parties, n_parties, device)
        self.root = root_dir
        for p in self.parties:
            if not os.path.isdir(os.path.join(root_dir, f"party{p}")):
                raise FileNotFoundError(f"no preprocessing directory {root_dir}/party{p}")

    def _take(self, key: MaterialKey, count: int):
        if key not in self._arrays:
            per, cnt = [], None
            for p in self.parties:
                path = os.path.join(self.root, f"party{p}", key.name() + ".bin")
                if not os.path.exists(path):
                    raise PreprocessingExhausted(f"party {p}: missing material file {path}")
                fkey, fparty, fn, c, arrays = read_material_file(path)
                if fkey != key or fparty != p or fn != self.n_parties:
                    raise ValueError(f"{path}: header does not match its name, party or n")
                cnt = c if cnt is None else cnt
                if c != cnt:
                    raise ValueError(f"{path}: count differs between parties")
                per.append(arrays)
            self.add_material(key, cnt, import_arrays(key, cnt, per, self.device))
        return super()._take(key, count)


def dealer_generate(seed: int, n_parties: int, demands: dict, out_dir: str, device="cuda") -> None:
    """On-device dealer -> per-party files + nothing else (preprocessing.py:232-243);
    byte-identical to the reference's files for the same seed and demand."""
    for p in range(n_parties):
        os.makedirs(os.path.join(out_dir, f"party{p}"), exist_ok=True)
    dealer = Dealer(seed, n_parties, 0, n_parties, device)
    for key, count in sorted(demands.items(), key=lambda kv: kv[0].name()):
        if count <= 0:
            continue
        arrays = dealer.generate(key, count, need_bits=True)
        for p in range(n_parties):
            write_material_file(os.path.join(out_dir, f"party{p}", key.name() + ".bin"), key, p, n_parties,
                                count, export_arrays(key, count, arrays, p))
