"""MPFXPRE1 dealer files (reference preprocessing.py:181-256).

CPU: files written by the reference's own dealer_generate parse and re-write
byte-identically; manifests round-trip. GPU: the on-device dealer writes
byte-identical files, and a FileStore over the reference's files drives the
B200 protocols to the golden (reference) output shares.
"""

import filecmp
import json
import os
import tempfile

import numpy as np
import pytest
import torch

from paper_2402_02320_b200 import material_io as mio

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = os.path.join(GOLDEN, "files")
CASES_WITH_FILES = {"reciprocal": 2, "batch_matmul": 3}


def _files(case):
    root = os.path.join(FILES, case)
    for p in range(CASES_WITH_FILES[case]):
        d = os.path.join(root, f"party{p}")
        for f in sorted(os.listdir(d)):
            yield p, os.path.join(d, f)


@pytest.mark.parametrize("case", sorted(CASES_WITH_FILES))
def test_reference_files_roundtrip_bytes(case):
    with tempfile.TemporaryDirectory() as tmp:
        for p, path in _files(case):
            key, party, n, count, arrays = mio.read_material_file(path)
            assert party == p and n == CASES_WITH_FILES[case]
            assert os.path.basename(path) == key.name() + ".bin"
            out = os.path.join(tmp, os.path.basename(path))
            mio.write_material_file(out, key, party, n, count, arrays)
            assert filecmp.cmp(path, out, shallow=False)


def test_manifest_roundtrip_and_rejects_garbage():
    man = mio.read_manifest(os.path.join(FILES, "reciprocal", "manifest.json"))
    with tempfile.TemporaryDirectory() as tmp:
        out = os.path.join(tmp, "m.json")
        mio.write_manifest(out, man)
        assert json.load(open(out)) == json.load(open(os.path.join(FILES, "reciprocal", "manifest.json")))
        bad = os.path.join(tmp, "bad.bin")
        open(bad, "wb").write(b"NOTAFILE" + bytes(40))
        with pytest.raises(ValueError):
            mio.read_material_file(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES_WITH_FILES))
def test_device_dealer_writes_reference_identical_files(case):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    demands = mio.read_manifest(os.path.join(FILES, case, "manifest.json"))
    with tempfile.TemporaryDirectory() as tmp:
        mio.dealer_generate(11, CASES_WITH_FILES[case], demands, tmp)
        for p, path in _files(case):
            mine = os.path.join(tmp, f"party{p}", os.path.basename(path))
            assert filecmp.cmp(path, mine, shallow=False), mine


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES_WITH_FILES))
def test_filestore_of_reference_files_reproduces_golden(case):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from cases import CASES
    from gpu_engine import GpuEngine
    from paper_2402_02320_b200.session import SimSession
    fn, n = CASES[case]
    store = mio.FileStore(os.path.join(FILES, case), tuple(range(n)), n)
    out = fn(GpuEngine(), SimSession(n, store))
    torch.cuda.synchronize()
    z = np.load(os.path.join(GOLDEN, f"{case}.npz"))
    for k, v in out.items():
        assert np.array_equal(GpuEngine.export(v), z[f"out__{k}"]), k
