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


def test_int32_index_boundary():
    """Node indices are int32 on the device (site * LPT + position).  C5
    (2160 x 3827 sites x 256 labels, 2.12e9 node slots) fits; 4096-wide 4K at
    256 labels (2.26e9) is refused with GZ_ERR_OVERFLOW instead of wrapping."""
    import ctypes as C
    L = _lib.lib()
    assert L.gz_workspace_bytes(2160, 3827, 256) > 100 * 2**30
    assert L.gz_workspace_bytes(2160, 4096, 256) == 0
    assert L.gz_workspace_bytes(65536, 32768, 2) == 0          # 2^31 sites x 16 lanes
    en = _lib.Energy(14, 1023, 0)
    sc = _lib.Sched(12, 0, 0, 0)
    st = _lib.Stats()
    p = C.c_void_p(16)
    assert L.gz_solve_volume(p, 2160, 4096, 256, C.byref(en), C.byref(sc), None, None, p, C.byref(st), p,
                             1 << 62, None) == _lib.GZ_ERR_OVERFLOW
    assert L.gz_solve_volume_batch(p, 2160, 4096, 256, C.byref(en), 1, C.byref(sc), p, C.byref(st), p, 1 << 62,
                                   None) == _lib.GZ_ERR_OVERFLOW
    devs = (C.c_int32 * 1)(0)
    assert L.gz_solve_volume_banded(p, 2160, 4096, 256, C.byref(en), C.byref(sc), None, None, 1, devs, p,
                                    C.byref(st)) == _lib.GZ_ERR_OVERFLOW
    cub = _lib.Cuboid(4610, 2160, -2304, 4096, 0, 2160, 2000, 256)
    assert L.gz_solve_pairs(p, p, 1, 2160, 4610, 3, C.byref(cub), C.byref(en), C.byref(sc), p, C.byref(st), p,
                            1 << 62, None) == _lib.GZ_ERR_OVERFLOW


def test_cuboid_wider_than_image_is_rejected():
    """k_sad clamps columns to width-1 but strides rows by the image width: a
    cuboid wider than the image is an argument error (IndexError upstream)."""
    import ctypes as C
    L = _lib.lib()
    cub = _lib.Cuboid(400, 288, -186, 372, 0, 288, 175, 16)
    p = C.c_void_p(16)
    assert L.gz_sad_volume(p, p, 288, 384, 3, C.byref(cub), p, None) == _lib.GZ_ERR_ARG
    en = _lib.Energy(14, 1023, 0)
    sc = _lib.Sched(12, 0, 0, 0)
    st = _lib.Stats()
    assert L.gz_solve_pairs(p, p, 1, 288, 384, 3, C.byref(cub), C.byref(en), C.byref(sc), p, C.byref(st), p,
                            1 << 30, None) == _lib.GZ_ERR_ARG
    # thin_skin: the coarse grid must cover the fine one
    assert L.gz_thin_skin(p, 10, 10, 31, 20, 16, 3, 1, p, p, None) == _lib.GZ_ERR_ARG


def test_stats_struct_matches_header():
    """ctypes Stats mirrors gz_stats field for field (new fields append)."""
    text = (ROOT / "include" / "gazecut_b200.h").read_text()
    body = text[text.index("typedef struct {\n    int64_t flow"):]
    body = body[: body.index("} gz_stats;")]
    names = re.findall(r"\b([a-z_][a-z_0-9]*)(?:\[\d+\])?\s*[,;]", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert names == [f[0] for f in _lib.Stats._fields_]


def test_explicit_network_entry_points_reject_bad_arguments():
    """The explicit-network C ABI (gz_csr.cuh) validates before any device work."""
    import ctypes as C
    L = _lib.lib()
    p = C.c_void_p(16)
    st = _lib.CsrStats()
    info = (C.c_int64 * 4)()
    en = _lib.Energy(14, 1023, 0)
    # export: missing volume (capacity mode), bad windows pairing, m > 256
    assert L.gz_export_arcs(None, 4, 5, 4, C.byref(en), None, None, 0, None, None, None, None, 0, info, p, 1 << 30,
                            None) == _lib.GZ_ERR_ARG
    assert L.gz_export_arcs(p, 4, 5, 4, C.byref(en), p, None, 0, None, None, None, None, 0, info, p, 1 << 30,
                            None) == _lib.GZ_ERR_ARG
    assert L.gz_export_arcs(p, 4, 5, 300, C.byref(en), None, None, 0, None, None, None, None, 0, info, p, 1 << 30,
                            None) == _lib.GZ_ERR_ARG
    assert L.gz_export_state(None, 4, 5, 4, 0, p, None) == _lib.GZ_ERR_ARG
    assert L.gz_export_state(p, 4, 5, 4, 99, p, None) == _lib.GZ_ERR_ARG
    # CSR max-flow: source == sink, out-of-range terminals, zero rounds, small workspace
    args = lambda n, s, t, rounds, ws: L.gz_maxflow_csr(n, s, t, p, p, p, p, p, rounds, -1, None, None,  # noqa: E731
                                                         C.byref(st), p, ws, None)
    assert args(10, 3, 3, 12, 1 << 30) == _lib.GZ_ERR_ARG
    assert args(10, 0, 10, 12, 1 << 30) == _lib.GZ_ERR_ARG
    assert args(10, 0, 9, 0, 1 << 30) == _lib.GZ_ERR_ARG
    assert args(10, 0, 9, 12, 16) == _lib.GZ_ERR_WORKSPACE
    assert L.gz_csr_workspace_bytes(1) == 0 and L.gz_csr_workspace_bytes(1000) > 8000
    assert L.gz_source_side_csr(10, 10, p, p, p, p, None) == _lib.GZ_ERR_ARG
    assert L.gz_chain_presaturate_csr(None, p, p, p, 4, p, None) == _lib.GZ_ERR_ARG
    assert L.gz_conservation_violations_csr(p, p, None, 4, 0, 3, p, None) == _lib.GZ_ERR_ARG
    # batched-pair workspace: invalid shapes size to 0 (no device query needed)
    assert L.gz_pairs_workspace_bytes(0, 5, 16, 8) == 0 and L.gz_pairs_workspace_bytes(4, 5, 1, 8) == 0
