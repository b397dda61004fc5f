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


def test_cpp_mirror_compiles_and_runs(tmp_path):
    """include/lightcache.hpp (stagecache-style C++ API over the C-ABI) links
    against liblightcache.so and maps status codes to the reference's
    exception types."""
    import os
    import subprocess
    root = lc.REPO_ROOT
    exe = str(tmp_path / "demo")
    libdir = os.path.dirname(lc.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-I" + os.path.join(root, "include"),
                    os.path.join(root, "tools", "cpp", "host_api_demo.cpp"), "-L" + libdir, "-llightcache",
                    "-Wl,-rpath," + libdir, "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    assert out.splitlines()[0].split() == ["F+", "c", "c!", "F+", "c", "c!", "F"]
    assert "ConfigError: unknown config key" in out


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lc.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
