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


def test_argument_errors_without_a_gpu():
    """Bad arguments are rejected before any device work (ValueError in the
    reference: energy.py:94-95, flownet.py:248-249, maxflow.py:418-419)."""
    import ctypes as C
    L = _lib.lib()
    cub = _lib.Cuboid(384, 288, -186, 372, 0, 288, 175, 16)
    en = _lib.Energy(14, 1023, 0)
    sc = _lib.Sched(12, 0, 0, 0)
    st = _lib.Stats()
    p = C.c_void_p(16)   # never dereferenced: argument checks come first
    # data term: null inputs, zero channels, rows outside the image
    assert L.gz_sad_volume(None, p, 288, 384, 3, C.byref(cub), p, None) == _lib.GZ_ERR_ARG
    assert L.gz_sad_volume(p, p, 288, 384, 0, C.byref(cub), p, None) == _lib.GZ_ERR_ARG
    bad = _lib.Cuboid(384, 288, -186, 372, 10, 288, 175, 16)
    assert L.gz_sad_volume(p, p, 288, 384, 3, C.byref(bad), p, None) == _lib.GZ_ERR_ARG
    # solve: empty grid, one window bound without the other, negative penalty, small workspace
    assert L.gz_solve_volume(p, 0, 5, 4, C.byref(en), C.byref(sc), None, None, p, C.byref(st), p, 1 << 30,
                             None) == _lib.GZ_ERR_ARG
    assert L.gz_solve_volume(p, 4, 5, 4, C.byref(en), C.byref(sc), p, None, p, C.byref(st), p, 1 << 30,
                             None) == _lib.GZ_ERR_ARG
    neg = _lib.Energy(-1, 5, 0)
    assert L.gz_solve_volume(p, 4, 5, 4, C.byref(neg), C.byref(sc), None, None, p, C.byref(st), p, 1 << 30,
                             None) == _lib.GZ_ERR_ARG
    assert L.gz_solve_volume(p, 4, 5, 4, C.byref(en), C.byref(sc), None, None, p, C.byref(st), p, 16,
                             None) == _lib.GZ_ERR_WORKSPACE
    # pairs: a single label cannot form a chain
    one = _lib.Cuboid(384, 288, -186, 372, 0, 288, 175, 1)
    assert L.gz_solve_pairs(p, p, 1, 288, 384, 3, C.byref(one), C.byref(en), C.byref(sc), p, C.byref(st), p,
                            1 << 30, None) == _lib.GZ_ERR_ARG
