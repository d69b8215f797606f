"""The C-ABI library loads without a GPU and exports every symbol the header declares."""

import ctypes
import re
from pathlib import Path

from paper_1803_01516_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "gazecut_b200.h").read_text()
    return sorted(set(re.findall(r"\b(gz_[a-z_0-9]+)\s*\(", text)))


def test_header_lists_match():
    assert declared() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared():
        assert hasattr(lib, name), name


def test_status_strings_and_workspace_sizing():
    L = _lib.lib()
    assert L.gz_status_string(0) == b"ok"
    assert b"energy" in L.gz_status_string(_lib.GZ_ERR_CONSISTENCY)
    assert L.gz_workspace_bytes(0, 5, 5) == 0
    small, big = L.gz_workspace_bytes(288, 372, 16), L.gz_workspace_bytes(288, 372, 24)
    assert 0 < small < big
    assert b"sm_100a" in L.gz_build_info()
