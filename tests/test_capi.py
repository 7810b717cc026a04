"""The C-ABI library builds/loads on CPU, exports every symbol include/p3d.h
declares, and its struct layouts match the ctypes mirrors (no compute calls)."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "p3d.h")
LIB = os.path.join(ROOT, "paper_2403_09070_b200", "libp3d.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t|void|double)\s+(p3d_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2403_09070_b200 import build

        build.build()
    from paper_2403_09070_b200 import _lib

    return _lib.load()


def test_exports_match_header(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r"\bT (p3d_\w+)$", out, flags=re.M)))
    decl = declared()
    assert decl, "no declarations parsed"
    assert set(decl) <= set(exported), set(decl) - set(exported)
    from paper_2403_09070_b200 import _lib

    assert set(_lib.EXPORTS) <= set(decl), set(_lib.EXPORTS) - set(decl)


def test_struct_sizes_and_version(lib):
    assert lib.p3d_abi_version() == 1
    # _lib.load() already asserted every sizeof matches the ctypes mirror


def test_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_path_without_gpu(lib):
    import ctypes as C

    from paper_2403_09070_b200 import _lib

    # a NULL topology is rejected before any CUDA call
    rc = lib.p3d_netboxes(None, None, None, None, None, None, None, None, None, None, None, None)
    assert rc == 1
    buf = C.create_string_buffer(256)
    assert lib.p3d_last_error(buf, 256) > 0 and b"topology" in buf.value
    with pytest.raises(ValueError):
        _lib.call("p3d_precondition", -1, None, 0.0, None, None, None, None, None, None)
