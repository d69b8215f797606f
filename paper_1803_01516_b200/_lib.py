"""ctypes binding of libgazecut_b200.so (the C ABI in include/gazecut_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1803_01516_b200.build``).  There is no fallback: if the
library or an sm_100 GPU is missing, every solver entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["GZ_LIB_PATH"]) if os.environ.get("GZ_LIB_PATH") else PKG_DIR / "libgazecut_b200.so"   # (A/B runs)

GZ_OK = 0
GZ_ERR_ARG = -1
GZ_ERR_CUDA = -2
GZ_ERR_WORKSPACE = -3
GZ_ERR_CONSISTENCY = -4
GZ_ERR_OVERFLOW = -5
GZ_ERR_NOCONVERGE = -6
GZ_ERR_NOGPU = -7
GZ_ERR_BANDS = -8
GZ_SCHED_NO_WAVE = 1
GZ_SCHED_CAPPED = 2
GZ_SCHED_V1 = 4
GZ_SCHED_V2 = 8   # retired (maps to the default v4 solver)
GZ_SCHED_V3 = 16  # retired (maps to the default v4 solver)
GZ_SCHED_INIT_ONLY = 32
# gz_export_state planes (include/gazecut_b200.h enum gz_plane)
GZ_PLANE_CHAIN, GZ_PLANE_SAME_RIGHT, GZ_PLANE_SAME_DOWN, GZ_PLANE_DIAG_RIGHT, GZ_PLANE_DIAG_LEFT, \
    GZ_PLANE_DIAG_DOWN, GZ_PLANE_DIAG_UP, GZ_PLANE_EXCESS, GZ_PLANE_HEIGHT = range(9)


class Cuboid(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("width", "height", "g_min", "g_extent", "y_min", "y_extent", "d_min", "m")]


class Gaze(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("g_min", "y_min", "d_min", "rows", "cols", "m", "offset1", "offset2", "offset3",
                 "lw_offset", "rw_offset", "h_offset")]


class Energy(C.Structure):
    _fields_ = [("penalty", C.c_int32), ("inhibit", C.c_int32), ("hard_inhibit", C.c_int32)]


class Sched(C.Structure):
    _fields_ = [("rounds_per_sweep", C.c_int32), ("max_sweeps", C.c_int32),
                ("bfs_cap", C.c_int32), ("flags", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("flow", "energy", "const_offset", "nodes", "arcs", "presaturated", "pushes",
                 "relabels", "labeling_energy", "node_updates")] + \
               [(n, C.c_int32) for n in
                ("sweeps", "converged", "stranded_excess_nodes", "bfs_passes", "reach_passes",
                 "pulses", "bfs_h", "excess_nodes")] + \
               [("ms_total", C.c_float), ("ms_phase", C.c_float * 6)]


class CsrStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("flow", "pushes", "relabels", "stranded_excess_nodes")] + \
               [(n, C.c_int32) for n in ("sweeps", "converged", "pulses")] + [("ms_total", C.c_float)]


class GazecutError(RuntimeError):
    """A device-side failure reported through the C ABI."""

    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


_LIB = None
_vp = C.c_void_p
_i32 = C.c_int32


def lib():
    """Load the shared library (raises OSError if it has not been built)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise OSError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        L.gz_workspace_bytes.restype = C.c_size_t
        L.gz_workspace_bytes.argtypes = [_i32, _i32, _i32]
        L.gz_sad_volume.restype = C.c_int
        L.gz_sad_volume.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Cuboid), _vp, _vp]
        L.gz_solve_volume.restype = C.c_int
        L.gz_solve_volume.argtypes = [_vp, _i32, _i32, _i32, C.POINTER(Energy), C.POINTER(Sched),
                                      _vp, _vp, _vp, C.POINTER(Stats), _vp, C.c_size_t, _vp]
        L.gz_solve_pairs.restype = C.c_int
        L.gz_solve_pairs.argtypes = [_vp, _vp, _i32, _i32, _i32, _i32, C.POINTER(Cuboid),
                                     C.POINTER(Energy), C.POINTER(Sched), _vp, C.POINTER(Stats),
                                     _vp, C.c_size_t, _vp]
        L.gz_pairs_workspace_bytes.restype = C.c_size_t
        L.gz_pairs_workspace_bytes.argtypes = [_i32, _i32, _i32, _i32]
        L.gz_pairs_launches.restype = C.c_int
        L.gz_pairs_launches.argtypes = [_i32, _i32, _i32, _i32, C.c_size_t]
        L.gz_solve_pairs_host.restype = C.c_int
        L.gz_solve_pairs_host.argtypes = L.gz_solve_pairs.argtypes
        L.gz_solve_volume_banded.restype = C.c_int
        L.gz_solve_volume_banded.argtypes = [_vp, _i32, _i32, _i32, C.POINTER(Energy), C.POINTER(Sched),
                                             _vp, _vp, _i32, _vp, _vp, C.POINTER(Stats)]
        L.gz_ground_truth_to_depth.restype = C.c_int
        L.gz_ground_truth_to_depth.argtypes = [_vp, _i32, _i32, _i32, C.POINTER(Gaze), _vp, _vp, _vp, _vp]
        L.gz_render_disparity.restype = C.c_int
        L.gz_render_disparity.argtypes = [_vp, C.POINTER(Gaze), _i32, _i32, _i32, _vp, _vp, _vp]
        L.gz_error_count.restype = C.c_int
        L.gz_error_count.argtypes = [_vp, _i32, _vp, _vp, _i32, _i32, _i32, _vp, _vp]
        L.gz_solve_volume_batch.restype = C.c_int
        L.gz_solve_volume_batch.argtypes = [_vp, _i32, _i32, _i32, _vp, _i32, C.POINTER(Sched), _vp, _vp,
                                            _vp, C.c_size_t, _vp]
        L.gz_total_energy.restype = C.c_int
        L.gz_total_energy.argtypes = [_vp, _vp, _i32, _i32, _i32, C.POINTER(Energy), _vp, _vp]
        L.gz_coarsen.restype = C.c_int
        L.gz_coarsen.argtypes = [_vp, _i32, _i32, _i32, _i32, _vp, _vp]
        L.gz_thin_skin.restype = C.c_int
        L.gz_thin_skin.argtypes = [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp]
        _i64 = C.c_int64
        L.gz_export_arcs.restype = C.c_int
        L.gz_export_arcs.argtypes = [_vp, _i32, _i32, _i32, C.POINTER(Energy), _vp, _vp, _i32, _vp, _vp, _vp, _vp,
                                     _i64, _vp, _vp, C.c_size_t, _vp]
        L.gz_export_state.restype = C.c_int
        L.gz_export_state.argtypes = [_vp, _i32, _i32, _i32, _i32, _vp, _vp]
        L.gz_csr_workspace_bytes.restype = C.c_size_t
        L.gz_csr_workspace_bytes.argtypes = [_i64]
        L.gz_maxflow_csr.restype = C.c_int
        L.gz_maxflow_csr.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp,
                                     C.POINTER(CsrStats), _vp, C.c_size_t, _vp]
        L.gz_source_side_csr.restype = C.c_int
        L.gz_source_side_csr.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, _vp]
        L.gz_chain_presaturate_csr.restype = C.c_int
        L.gz_chain_presaturate_csr.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp]
        L.gz_conservation_violations_csr.restype = C.c_int
        L.gz_conservation_violations_csr.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp]
        L.gz_status_string.restype = C.c_char_p
        L.gz_status_string.argtypes = [C.c_int]
        L.gz_build_info.restype = C.c_char_p
        _LIB = L
    return _LIB


def status_string(status: int) -> str:
    try:
        return lib().gz_status_string(int(status)).decode()
    except OSError:
        return f"status {status}"


def check(status: int, where: str) -> None:
    if status != GZ_OK:
        raise GazecutError(status, where)


# Every symbol include/gazecut_b200.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "gz_workspace_bytes", "gz_sad_volume", "gz_solve_volume", "gz_solve_pairs", "gz_pairs_workspace_bytes", "gz_pairs_launches",
    "gz_solve_pairs_host", "gz_solve_volume_banded", "gz_ground_truth_to_depth",
    "gz_error_count", "gz_render_disparity", "gz_solve_volume_batch", "gz_total_energy", "gz_coarsen", "gz_thin_skin",
    "gz_status_string", "gz_build_info", "gz_export_arcs", "gz_export_state", "gz_csr_workspace_bytes",
    "gz_maxflow_csr", "gz_source_side_csr", "gz_chain_presaturate_csr", "gz_conservation_violations_csr",
)
