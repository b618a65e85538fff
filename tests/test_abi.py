"""The C-ABI boundary (include/mpx.h <-> libmpx.so <-> the Python bindings).

CPU: the library loads and exports every declared symbol; every prototype's
arity and argument kinds match the ctypes argtypes the package binds
(``_lib._SIGS`` / ``_PLAIN`` and the fused-kernel bindings in ``fused.py``)
and the reference-side stub in INTEGRATION.md §2; precondition failures
return MPX_ERR_ARG without touching a GPU and map to ``MpxError``.
GPU: the INTEGRATION.md stub runs and equals numpy's wrapping uint64 matmul
(the reference's ring.matmul, ring.py:60-62).
"""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2402_02320_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "mpx.h")


def prototypes() -> dict:
    """name -> (return type, [parameter types]) for every mpx_* declaration."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    out = {}
    for ret, name, params in re.findall(r"^(int|const char\s*\*)\s+(mpx_\w+)\s*\(([^)]*)\)\s*;", src, flags=re.M):
        ps = [p.strip() for p in params.replace("\n", " ").split(",") if p.strip() and p.strip() != "void"]
        types = []
        for p in ps:
            p = re.sub(r"\s+", " ", p)
            t = p.rsplit(" ", 1)[0] if "*" not in p.rsplit(" ", 1)[-1] else p
            types.append("ptr" if "*" in p else t.replace("const ", "").strip())
        out[name] = (ret.replace(" ", ""), types)
    return out


_KIND = {ctypes.c_void_p: "ptr", ctypes.c_int64: "int64_t", ctypes.c_uint64: "uint64_t", ctypes.c_int: "int",
         ctypes.c_char_p: "ptr"}


def _kind(ct):
    if ct in _KIND:
        return _KIND[ct]
    if isinstance(ct, type) and issubclass(ct, ctypes._Pointer):
        return "ptr"
    raise AssertionError(f"unexpected ctypes type {ct}")


def declared():
    return sorted(prototypes())


def test_header_declares_the_abi():
    names = declared()
    assert len(names) >= 40
    assert set(names) == set(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    assert _lib.version().startswith("libmpx")


def test_elf_dynamic_symbols():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def _normalise(t):
    return {"size_t": "int64_t", "long long": "int64_t"}.get(t, t)


def test_every_binding_matches_its_prototype():
    from paper_2402_02320_b200 import fused
    lib = _lib.load()
    fused._bind()
    protos = prototypes()
    for name, (ret, params) in protos.items():
        fn = getattr(lib, name)
        assert fn.argtypes is not None, f"{name} is never bound"
        got = [_kind(a) for a in fn.argtypes]
        assert got == [_normalise(p) for p in params], (name, got, params)
        assert (fn.restype is ctypes.c_char_p) == (ret == "constchar*"), name
    # every stream-taking entry ends with the stream (call() appends it)
    for name, args in _lib._SIGS.items():
        assert protos[name][1][-1] == "ptr" and len(args) == len(protos[name][1]), name


def test_integration_stub_matches_header():
    """INTEGRATION.md §2's reference-side ctypes block binds the header's arity."""
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# mpfix/_b200\.py.*?)```", text, flags=re.S).group(1)
    block = block.replace('"/path/to/paper_2402_02320_b200/libmpx.so"', repr(_lib.LIB_PATH))
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    protos = prototypes()
    for name in ("mpx_limb_split", "mpx_gemm_limbs"):
        got = [_kind(a) for a in getattr(ns["lib"], name).argtypes]
        assert got == [_normalise(p) for p in protos[name][1]], name


def test_argument_errors_return_mpx_err_arg_and_raise():
    """CHECK_ARG runs before any CUDA call: safe without a GPU."""
    lib = _lib.load()
    assert lib.mpx_encode(None, None, 10, 64, 23, None) == _lib.MPX_ERR_ARG
    assert lib.mpx_encode(None, None, 10, 65, 23, None) == _lib.MPX_ERR_ARG
    assert lib.mpx_ring_mul(None, None, None, -1, 64, None) == _lib.MPX_ERR_ARG
    with pytest.raises(_lib.MpxError, match="invalid argument"):
        _lib.check("mpx_encode", lib.mpx_encode(None, None, 10, 64, 23, None))
    _lib.check("mpx_encode", _lib.MPX_OK)


@pytest.mark.gpu
def test_integration_stub_runs_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# mpfix/_b200\.py.*?)```", text, flags=re.S).group(1)
    block = block.replace('"/path/to/paper_2402_02320_b200/libmpx.so"', repr(_lib.LIB_PATH))
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(3)
    for m, k, r in ((256, 384, 96), (200, 1000, 77)):
        a = rng.integers(0, 1 << 64, (m, k), dtype=np.uint64)
        b = rng.integers(0, 1 << 64, (k, r), dtype=np.uint64)
        assert np.array_equal(ns["ring_matmul_b200"](a, b, 64), np.matmul(a, b))
    assert _lib.device_sm_count() == torch.cuda.get_device_properties(0).multi_processor_count
