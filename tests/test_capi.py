"""The C-ABI library loads without a GPU and exports every symbol that
include/lightcache.h declares (no compute calls here)."""
import ctypes
import re

import paper_2510_05367_b200 as lc


def _declared():
    src = open(lc.HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(lc_[a-z0-9_]+)\s*\(", src)))


def test_header_and_exports_agree():
    assert _declared() == sorted(lc.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = lc.lib()
    for name in _declared():
        assert isinstance(getattr(L, name), ctypes._CFuncPtr), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
