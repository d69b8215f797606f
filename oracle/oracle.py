"""ctypes front end of the CPU oracle (oracle/gz_oracle.c) plus the small
numpy restatements of the reference's host-side helpers.

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg, never by the shipped
package.  Every function cites the reference routine it restates (paths under
/root/reference/pkg/src/gazecut/).  Parity of this oracle with the reference
is pinned in tests/test_oracle.py against the reference's own golden vectors
and against fixtures produced by running the reference (oracle/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libgz_oracle.so"
UNCUTTABLE = 1 << 56  # energy.py:34

_i64 = C.c_int64
_p = C.c_void_p


class _Net(C.Structure):
    _fields_ = [
        ("n_nodes", _i64), ("source", _i64), ("sink", _i64), ("n_arcs", _i64),
        ("const_offset", _i64), ("rows", _i64), ("cols", _i64), ("m", _i64),
        ("n_chain", _i64),
        ("first_out", _p), ("head", _p), ("rev", _p), ("cap", _p), ("resid", _p),
        ("lo", _p), ("hi", _p), ("node_base", _p), ("chain_arcs", _p), ("chain_base", _p),
    ]


class _PRStats(C.Structure):
    _fields_ = [
        ("flow", _i64), ("presaturated", _i64), ("pushes", _i64), ("relabels", _i64),
        ("stranded", _i64), ("sweeps", C.c_int32), ("converged", C.c_int32),
    ]


def build_lib(force: bool = False) -> Path:
    """Compile gz_oracle.c with gcc (no GPU, no reference needed)."""
    srcs = [HERE / "gz_oracle.c", HERE / "gz_certify.c", HERE / "gz_capped.c"]
    if force or not LIB_PATH.exists() or any(LIB_PATH.stat().st_mtime < s.stat().st_mtime for s in srcs):
        subprocess.run(
            ["gcc", "-O2", "-shared", "-fPIC", "-std=c11", "-o", str(LIB_PATH), *map(str, srcs)],
            check=True,
        )
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        build_lib()
        L = C.CDLL(str(LIB_PATH))
        L.gzo_build_network.restype = C.POINTER(_Net)
        L.gzo_build_network.argtypes = [_p, _i64, _i64, _i64, _i64, _i64, _p, _p]
        L.gzo_network_from_arcs.restype = C.POINTER(_Net)
        L.gzo_network_from_arcs.argtypes = [_i64, _i64, _i64, _i64, _p, _p, _p, _p]
        L.gzo_free.argtypes = [C.POINTER(_Net)]
        L.gzo_reset.argtypes = [C.POINTER(_Net)]
        L.gzo_maxflow_dinic.restype = _i64
        L.gzo_maxflow_dinic.argtypes = [C.POINTER(_Net)]
        L.gzo_maxflow_push_relabel.restype = C.c_int
        L.gzo_maxflow_push_relabel.argtypes = [
            C.POINTER(_Net), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_PRStats)]
        L.gzo_chain_presaturate.restype = _i64
        L.gzo_chain_presaturate.argtypes = [C.POINTER(_Net)]
        L.gzo_source_side.argtypes = [C.POINTER(_Net), _p]
        L.gzo_extract_labels.restype = _i64
        L.gzo_extract_labels.argtypes = [C.POINTER(_Net), _p, _p]
        L.gzo_conservation_violations.restype = _i64
        L.gzo_conservation_violations.argtypes = [C.POINTER(_Net)]
        L.gzo_node_blocks.argtypes = [C.POINTER(_Net), _i64, _p]
        L.gzo_total_energy.restype = _i64
        L.gzo_total_energy.argtypes = [_p, _p, C.c_int, C.c_int, C.c_int, _i64, _i64, C.c_int]
        L.gzo_sad_volume.argtypes = [_p, _p] + [C.c_int] * 10 + [_p]
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _view(addr, n, dtype):
    if n == 0 or not addr:
        return np.empty(0, dtype=dtype)
    ct = {np.int64: C.c_int64, np.int32: C.c_int32}[dtype]
    return np.ctypeslib.as_array(C.cast(addr, C.POINTER(ct)), shape=(int(n),))


class OracleNet:
    """CSR flow network, same layout as the reference FlowNetwork (flownet.py:41-89)."""

    def __init__(self, handle):
        self._h = handle
        s = handle.contents
        self.n_nodes, self.source, self.sink = int(s.n_nodes), int(s.source), int(s.sink)
        self.num_arcs = int(s.n_arcs)
        self.const_offset = int(s.const_offset)
        self.site_shape = (int(s.rows), int(s.cols)) if s.rows else None
        self.num_labels = int(s.m) if s.rows else None
        n, a = self.n_nodes, self.num_arcs
        self.first_out = _view(s.first_out, n + 1, np.int64)
        self.head = _view(s.head, a, np.int32)
        self.rev = _view(s.rev, a, np.int32)
        self.cap = _view(s.cap, a, np.int64)
        self.resid = _view(s.resid, a, np.int64)
        if s.rows:
            sites = int(s.rows * s.cols)
            self.lo = _view(s.lo, sites, np.int32)
            self.hi = _view(s.hi, sites, np.int32)
            self.node_base = _view(s.node_base, sites + 1, np.int64)
            self.chain_arcs = _view(s.chain_arcs, int(s.n_chain), np.int32)
            self.chain_base = _view(s.chain_base, sites + 1, np.int64)

    def __del__(self):
        if getattr(self, "_h", None) is not None and _LIB is not None:
            _LIB.gzo_free(self._h)
            self._h = None

    def reset(self):
        lib().gzo_reset(self._h)

    def dump(self) -> str:
        """flownet.py:385-397 dump_network text format."""
        lines = [f"nodes {self.n_nodes} source {self.source} sink {self.sink} offset {self.const_offset}"]
        for u in range(self.n_nodes):
            for a in range(int(self.first_out[u]), int(self.first_out[u + 1])):
                lines.append(f"{u} {int(self.head[a])} {int(self.cap[a])}")
        return "\n".join(lines) + "\n"


def build_network(volume, penalty: int, inhibit_cap: int, lo=None, hi=None) -> OracleNet:
    """flownet.py:233-296."""
    vol = np.ascontiguousarray(volume, dtype=np.int64)
    rows, cols, m = vol.shape
    sites = rows * cols
    lo_a = hi_a = None
    if lo is not None and hi is not None:
        lo_a = np.ascontiguousarray(np.asarray(lo, dtype=np.int32).reshape(sites))
        hi_a = np.ascontiguousarray(np.asarray(hi, dtype=np.int32).reshape(sites))
    h = lib().gzo_build_network(
        _ptr(vol), rows, cols, m, int(penalty), int(inhibit_cap),
        _ptr(lo_a) if lo_a is not None else None, _ptr(hi_a) if hi_a is not None else None)
    if not h:
        raise ValueError("label windows must satisfy 0 <= lo <= hi < num_labels")
    return OracleNet(h)


def network_from_arcs(n_nodes, source, sink, arcs) -> OracleNet:
    """flownet.py:325-353."""
    k = len(arcs)
    pu = np.empty(k, np.int64); pv = np.empty(k, np.int64)
    pc = np.empty(k, np.int64); prc = np.zeros(k, np.int64)
    for i, arc in enumerate(arcs):
        u, v, c = arc[0], arc[1], arc[2]
        if not (0 <= u < n_nodes and 0 <= v < n_nodes):
            raise ValueError(f"arc ({u}, {v}) outside node range")
        if c < 0 or (len(arc) > 3 and arc[3] < 0):
            raise ValueError("negative capacity")
        pu[i], pv[i], pc[i] = u, v, c
        if len(arc) > 3:
            prc[i] = arc[3]
    return OracleNet(lib().gzo_network_from_arcs(n_nodes, source, sink, k, _ptr(pu), _ptr(pv), _ptr(pc), _ptr(prc)))


def node_blocks(net: OracleNet, block: int) -> np.ndarray:
    out = np.zeros(net.n_nodes, np.int32)
    lib().gzo_node_blocks(net._h, block, _ptr(out))
    return out


def source_side(net: OracleNet) -> np.ndarray:
    side = np.zeros(net.n_nodes, np.uint8)
    lib().gzo_source_side(net._h, _ptr(side))
    return side.astype(bool)


def extract_labeling(net: OracleNet, side=None) -> np.ndarray:
    if side is None:
        side = source_side(net)
    side_u8 = np.ascontiguousarray(side, dtype=np.uint8)
    rows, cols = net.site_shape
    labels = np.empty(rows * cols, np.int32)
    bad = lib().gzo_extract_labels(net._h, _ptr(side_u8), _ptr(labels))
    if bad:
        raise AssertionError(f"{bad} chains cut more than once")
    return labels.reshape(rows, cols)


def conservation_violations(net: OracleNet) -> int:
    return int(lib().gzo_conservation_violations(net._h))


def chain_presaturate(net: OracleNet) -> int:
    return int(lib().gzo_chain_presaturate(net._h))


def maxflow_push_relabel(net: OracleNet, rounds_per_sweep=12, max_sweeps=None, block=None, presaturate=True):
    """maxflow.py:403-478.  Returns (flow, energy-or-None, labeling, side, stats)."""
    if rounds_per_sweep < 1:
        raise ValueError("rounds_per_sweep must be >= 1")
    st = _PRStats()
    rc = lib().gzo_maxflow_push_relabel(
        net._h, int(rounds_per_sweep), -1 if max_sweeps is None else int(max_sweeps),
        0 if block is None else int(block), 1 if presaturate else 0, C.byref(st))
    if rc != 0:
        raise ValueError("push-relabel rejected its arguments")
    stats = {
        "solver": "push-relabel", "converged": bool(st.converged), "sweeps": int(st.sweeps),
        "pushes": int(st.pushes), "relabels": int(st.relabels),
        "presaturated": int(st.presaturated), "stranded_excess_nodes": int(st.stranded),
    }
    side = source_side(net)
    labeling = energy = None
    if net.site_shape is not None:
        labeling = extract_labeling(net, side)
        if st.converged:
            energy = int(st.flow) + net.const_offset
    return int(st.flow), energy, labeling, side, stats


def maxflow_dinic(net: OracleNet):
    """maxflow.py:385-400."""
    flow = int(lib().gzo_maxflow_dinic(net._h))
    side = source_side(net)
    labeling = energy = None
    if net.site_shape is not None:
        labeling = extract_labeling(net, side)
        energy = flow + net.const_offset
    return flow, energy, labeling, side, {"solver": "dinic", "converged": True}


def sad_volume(left, right, g_min, g_extent, y_min, y_extent, d_min, m, width=None) -> np.ndarray:
    """energy.py:83-114 (cuboid passed as its integer fields)."""
    left = np.ascontiguousarray(left, dtype=np.uint8)
    right = np.ascontiguousarray(right, dtype=np.uint8)
    if left.shape != right.shape:
        raise ValueError(f"image shapes differ: {left.shape} vs {right.shape}")
    if left.ndim == 2:
        left = left[:, :, None]
        right = right[:, :, None]
    h, w, ch = left.shape
    width = w if width is None else width
    vol = np.empty((y_extent, g_extent, m), np.int64)
    lib().gzo_sad_volume(_ptr(left), _ptr(right), h, w, ch, width, g_min, g_extent, y_min, y_extent,
                         d_min, m, _ptr(vol))
    return vol


def total_energy(labeling, volume, penalty, inhibit, hard=False) -> int:
    """energy.py:129-155."""
    lab = np.ascontiguousarray(labeling, dtype=np.int32)
    vol = np.ascontiguousarray(volume, dtype=np.int64)
    rows, cols, m = vol.shape
    if lab.shape != (rows, cols):
        raise ValueError("labeling shape mismatch")
    if lab.min() < 0 or lab.max() >= m:
        raise ValueError("label outside volume range")
    return int(lib().gzo_total_energy(_ptr(lab), _ptr(vol), rows, cols, m, int(penalty), int(inhibit),
                                      1 if hard else 0))


def solve_exact(volume, penalty, inhibit, hard=False, rounds_per_sweep=12, solver="push-relabel"):
    """maxflow.py:481-510 (identity check included)."""
    vol = np.ascontiguousarray(volume, dtype=np.int64)
    inhibit_cap = UNCUTTABLE if hard else inhibit
    net = build_network(vol, penalty, inhibit_cap)
    if solver == "push-relabel":
        flow, energy, lab, side, stats = maxflow_push_relabel(net, rounds_per_sweep)
    elif solver == "dinic":
        flow, energy, lab, side, stats = maxflow_dinic(net)
    else:
        raise ValueError(f"unknown solver {solver!r}")
    check = total_energy(lab, vol, penalty, inhibit, hard)
    if check != energy:
        raise AssertionError(f"cut cost {energy} != labeling energy {check}")
    stats.update(nodes=net.n_nodes, arcs=net.num_arcs, const_offset=net.const_offset)
    return {"flow": flow, "energy": energy, "labeling": lab, "source_side": side, "stats": stats}


def coarsen(volume, block, penalty):
    """hierarchy.py:39-57: zero-pad to multiples of ``block``, sum cubes, penalty * block."""
    if block < 1:
        raise ValueError("block must be >= 1")
    vol = np.asarray(volume, dtype=np.int64)
    r, c, m = vol.shape
    rb, cb, mb = -(-r // block), -(-c // block), -(-m // block)
    pad = np.zeros((rb * block, cb * block, mb * block), np.int64)
    pad[:r, :c, :m] = vol
    return pad.reshape(rb, block, cb, block, mb, block).sum(axis=(1, 3, 5)), penalty * block


def thin_skin(coarse_labeling, fine_shape, block, radius=1):
    """hierarchy.py:60-73."""
    rows, cols, m = fine_shape
    up = np.asarray(coarse_labeling, np.int64).repeat(block, 0).repeat(block, 1)[:rows, :cols]
    lo = np.maximum(block * (up - radius), 0)
    hi = np.minimum(block * (up + radius + 1) - 1, m - 1)
    return lo.astype(np.int32), hi.astype(np.int32)


def _restricted(vol, penalty, inhibit, hard, lo, hi, rounds):
    net = build_network(vol, penalty, UNCUTTABLE if hard else inhibit, lo, hi)
    flow, energy, lab, side, stats = maxflow_push_relabel(net, rounds)
    if total_energy(lab, vol, penalty, inhibit, hard) != energy:
        raise AssertionError("cut cost != labeling energy")
    return flow, energy, lab, net


def solve_level1(volume, penalty, inhibit, block, skin_radius=1, hard=False, rounds_per_sweep=12):
    """hierarchy.py:92-117."""
    vol = np.ascontiguousarray(volume, dtype=np.int64)
    cvol, cpen = coarsen(vol, block, penalty)
    _, ce, clab, _ = _restricted(cvol, cpen, inhibit, hard, None, None, rounds_per_sweep)
    lo, hi = thin_skin(clab, vol.shape, block, skin_radius)
    flow, energy, lab, net = _restricted(vol, penalty, inhibit, hard, lo, hi, rounds_per_sweep)
    return {"flow": flow, "energy": energy, "labeling": lab, "coarse_energy": ce,
            "coarse_labeling": clab, "lo": lo, "hi": hi, "const_offset": net.const_offset}


def solve_level2(volume, penalty, inhibit, block, skin_radius=1, hard=False, rounds_per_sweep=12,
                 max_sweeps=8):
    """hierarchy.py:120-165 (reference schedule: FIFO rounds in block order)."""
    vol = np.ascontiguousarray(volume, dtype=np.int64)
    cvol, cpen = coarsen(vol, block, penalty)
    _, ce, clab, _ = _restricted(cvol, cpen, inhibit, hard, None, None, rounds_per_sweep)
    lo, hi = thin_skin(clab, vol.shape, block, skin_radius)
    net = build_network(vol, penalty, UNCUTTABLE if hard else inhibit, lo, hi)
    flow, _, lab, _, stats = maxflow_push_relabel(net, rounds_per_sweep, max_sweeps, block)
    energy = total_energy(lab, vol, penalty, inhibit, hard)
    return {"flow": flow, "energy": energy, "labeling": lab, "coarse_energy": ce,
            "converged": stats["converged"], "lo": lo, "hi": hi, "const_offset": net.const_offset}


if os.environ.get("GZ_ORACLE_BUILD_ON_IMPORT"):
    build_lib()


# ---------------------------------------------------------------------------
# accuracy accounting (numpy restatements; test infrastructure only)

def _round_away_half(a):
    """geometry.py:37-47: halve, .5 away from zero."""
    return np.sign(a) * ((np.abs(a) + 1) // 2)


def ground_truth_to_depth(gt_image, scale, g_min, y_min, d_min, rows, cols, m, offset1, offset2, offset3,
                          lw_offset, rw_offset, h_offset):
    """imaging.py:155-201 -> (depth int32, valid bool, out_of_range, off_grid, collisions)."""
    gt = np.asarray(gt_image)
    ys, xs = np.nonzero(gt)
    dis = (gt[ys, xs].astype(np.int64) * 2 + scale) // (2 * scale)
    W = xs - _round_away_half(lw_offset + rw_offset) + _round_away_half(dis)
    S = _round_away_half(lw_offset - rw_offset) - _round_away_half(dis)
    gi = (W - offset1) - g_min
    yi = (ys - h_offset + offset2) - y_min
    k = (S - offset3) - d_min
    on_grid = (gi >= 0) & (gi < cols) & (yi >= 0) & (yi < rows)
    in_range = (k >= 0) & (k < m)
    keep = on_grid & in_range
    best = np.full((rows, cols), m, dtype=np.int64)
    np.minimum.at(best, (yi[keep], gi[keep]), k[keep])
    valid = best < m
    depth = np.where(valid, best, 0).astype(np.int32)
    return depth, valid, int((on_grid & ~in_range).sum()), int((~on_grid).sum()), int(keep.sum() - valid.sum())


def error_count(labeling, depth, valid, tail=9):
    """evalreport.py:47-61 -> (total_error, evaluated, histogram[0..tail])."""
    diff = np.abs(np.asarray(labeling, np.int64) - np.asarray(depth, np.int64))[np.asarray(valid, bool)]
    hist = np.bincount(np.minimum(diff, tail), minlength=tail + 1)
    return int(diff.sum()), int(diff.size), hist.astype(np.int64)


CERTIFY_CHECKS = {1: "capacity bounds", 2: "conservation", 3: "flow value", 4: "cut cost",
                  5: "minimal source side", 6: "out of memory"}


def certify(vol, penalty, inhibit, planes: dict, labels, device_flow):
    """oracle/gz_certify.c: the device state is a feasible maximum preflow whose
    value equals the labeling's cut cost, and the labeling is the minimal source
    side.  planes: int32 (P, m-1) arrays keyed cu, ph, pv,
    dar, dbr, dad, dbd, e.  Returns (failed check or 0, report dict)."""
    vol = np.ascontiguousarray(vol, dtype=np.int32)
    rows, cols, m = vol.shape
    arrs = [np.ascontiguousarray(planes[k], dtype=np.int32) for k in ("cu", "ph", "pv", "dar", "dbr", "dad", "dbd", "e")]
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    rep = np.zeros(8, np.int64)
    f = lib().gzc_certify
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, C.c_int, _p, C.c_int32, C.c_int32] + [_p] * 9 + [_i64, _p]
    rc = int(f(rows, cols, m, _ptr(vol), int(penalty), int(inhibit), *[_ptr(a) for a in arrs], _ptr(lab),
               int(device_flow), _ptr(rep)))
    keys = ("sink_inflow", "labeling_energy", "reached", "first_bad", "label_mismatches", "excess_nodes")
    return rc, dict(zip(keys, (int(x) for x in rep[:6])))


def capped_schedule(volume, penalty, inhibit, lo, hi, K, max_sweeps, bfs_min, H, presaturate=True):
    """oracle/gz_capped.c: the device's deterministic capped (level-2) schedule
    restated on the CPU.  Returns (labels (rows, cols) int32, report dict)."""
    vol = np.ascontiguousarray(volume, dtype=np.int32)
    rows, cols, m = vol.shape
    lo_a = np.ascontiguousarray(np.asarray(lo, dtype=np.int32).reshape(rows * cols))
    hi_a = np.ascontiguousarray(np.asarray(hi, dtype=np.int32).reshape(rows * cols))
    if int((hi_a - lo_a).max(initial=0)) > 63:
        raise ValueError("windows wider than 63 positions are not restated")
    lab = np.empty(rows * cols, np.int32)
    rep = np.zeros(4, np.int64)
    f = lib().gzo_capped
    f.restype = C.c_int
    f.argtypes = [_p, C.c_int, C.c_int, C.c_int, C.c_int32, C.c_int32, _p, _p, C.c_int, C.c_int, C.c_int, C.c_int,
                  C.c_int, _p, _p]
    f(_ptr(vol), rows, cols, m, int(penalty), int(inhibit), _ptr(lo_a), _ptr(hi_a), int(K), int(max_sweeps),
      int(bfs_min), int(H), 1 if presaturate else 0, _ptr(lab), _ptr(rep))
    return lab.reshape(rows, cols), dict(zip(("flow", "sweeps", "pulses", "converged"), (int(x) for x in rep)))
