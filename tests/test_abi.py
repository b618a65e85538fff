"""CPU: the C-ABI library loads and exports every symbol include/mpx.h declares
(no compute calls: there is no GPU here)."""

import ctypes
import os
import re

from paper_2402_02320_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "mpx.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(mpx_\w+)\(", src, flags=re.M)))


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
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name
