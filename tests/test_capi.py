"""The C-ABI library loads and exports every symbol include/potflow_b200.h declares
(no device calls: runs on CPU)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HDR = os.path.join(ROOT, "include", "potflow_b200.h")
LIB = os.path.join(ROOT, "paper_2601_05765_b200", "libpotflow_b200.so")


def declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_api():
    names = declared()
    for must in ("pf_batch_evaluate", "pf_grid_build", "pf_knn", "pf_dpsi_max", "pf_set_domain"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_exports_all_declared_symbols():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    lib.pf_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.pf_version()


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
