"""Max-flow / min-cut on the device and the cut read-out.

Mirrors ``gazecut.maxflow`` (maxflow.py:1-510).  ``maxflow_push_relabel``
runs the sm_100a push-relabel solver (gz_solve_volume); the labeling is the
canonical minimal source side of the minimum cut, identical to the one the
reference extracts (maxflow.py:1-16), so exact solves agree bit for bit.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _dev, _lib
from .energy import EnergyParams
from .flownet import FlowNetwork, build_network


@dataclass
class CutResult:
    """maxflow.py:34-48."""

    flow: int
    energy: Optional[int] = None
    labeling: Optional[np.ndarray] = None
    source_side: Optional[np.ndarray] = None
    stats: dict = field(default_factory=dict)


class InternalConsistencyError(AssertionError):
    """A solver invariant failed (maxflow.py:51-52)."""


def _sched(rounds_per_sweep: int, max_sweeps: Optional[int], presaturate: bool, bfs_cap: int) -> _lib.Sched:
    flags = 0 if presaturate else _lib.GZ_SCHED_NO_WAVE
    if max_sweeps is not None:
        flags |= _lib.GZ_SCHED_CAPPED
    return _lib.Sched(int(rounds_per_sweep), 0 if max_sweeps is None else max(int(max_sweeps), 0),
                      int(bfs_cap), flags)


def _run(net: FlowNetwork, rounds_per_sweep: int, max_sweeps: Optional[int], presaturate: bool,
         bfs_cap: int = 0) -> tuple[torch.Tensor, _lib.Stats]:
    rows, cols = net.site_shape
    m = net.num_labels
    L = _lib.lib()
    nbytes = L.gz_workspace_bytes(rows, cols, m)
    ws = _dev.workspace(nbytes)
    labels = torch.empty(rows * cols, dtype=torch.int32, device=net.volume.device)
    st = _lib.Stats()
    en = net.params._c()
    sc = _sched(rounds_per_sweep, max_sweeps, presaturate, bfs_cap)
    lo = _dev.ptr(net.lo) if net.lo is not None else None
    hi = _dev.ptr(net.hi) if net.hi is not None else None
    rc = L.gz_solve_volume(_dev.ptr(net.volume), rows, cols, m, C.byref(en), C.byref(sc), lo, hi,
                           _dev.ptr(labels), C.byref(st), _dev.ptr(ws), nbytes, _dev.stream_ptr())
    _lib.check(rc, "gz_solve_volume")
    return labels, st


def maxflow_push_relabel(net: FlowNetwork, rounds_per_sweep: int = 12, max_sweeps: Optional[int] = None,
                         block: Optional[int] = None, presaturate: bool = True) -> CutResult:
    """Preflow-push with global relabeling on the device (maxflow.py:403-478).

    ``max_sweeps`` caps the number of sweeps (global relabel + pulses): the
    level-2 approximation, ``stats['converged']`` False when the cap bit.
    ``block`` is accepted for API parity; the device schedule is the tile
    order of the implicit grid (level 2)."""
    if rounds_per_sweep < 1:
        raise ValueError("rounds_per_sweep must be >= 1")
    t0 = time.perf_counter()
    labels, st = _run(net, rounds_per_sweep, max_sweeps, presaturate)
    converged = bool(st.converged)
    wall = time.perf_counter() - t0
    if net.lo is None and net.const_offset != int(st.const_offset):
        raise InternalConsistencyError("device constant offset disagrees with the graph size model")
    net.labels_dev = labels
    stats = {
        "solver": "push-relabel",
        "wall_s": wall,
        "converged": converged,
        "sweeps": int(st.sweeps),
        "pushes": int(st.pushes),
        "relabels": int(st.relabels),
        "presaturated": int(st.presaturated),
        "stranded_excess_nodes": int(st.stranded_excess_nodes),
        "excess_nodes": int(st.excess_nodes),
        "bfs_h": int(st.bfs_h),
        "device": "sm_100a",
        "device_ms": float(st.ms_total),
        "pulses": int(st.pulses),
        "bfs_passes": int(st.bfs_passes),
        "reach_passes": int(st.reach_passes),
        "labeling_energy": int(st.labeling_energy),
        "node_updates": int(st.node_updates),
        "phase_ms": {k: round(float(v), 4) for k, v in
                     zip(("init", "mask_build", "global_relabel", "pulses", "extract", "tail"), st.ms_phase)},
    }
    if block is not None:
        stats["block"] = int(block)
    net.last_stats = stats
    flow = int(st.flow)
    result = CutResult(flow=flow, stats=stats)
    result.labeling = labels.view(net.site_shape).cpu().numpy()
    result.source_side = source_side(net)
    if converged:
        result.energy = flow + net.const_offset
    return result


def maxflow_reference(net: FlowNetwork) -> CutResult:
    """maxflow.py:385-400 names Dinic's algorithm.  The minimum cut read-out is
    canonical, so the device solver returns the identical flow and labeling;
    ``stats['solver']`` records what actually ran."""
    r = maxflow_push_relabel(net)
    r.stats["requested_solver"] = "dinic"
    return r


def source_side(net: FlowNetwork) -> np.ndarray:
    """maxflow.py:355-359: bool per node (chains site-major, source, sink).

    Chains are cut exactly once (uncuttable reverse arcs), so the source side
    of site s is chain positions lo+1 .. label: derived on the device."""
    if net.labels_dev is None:
        raise ValueError("network has not been solved")
    rows, cols = net.site_shape
    m = net.num_labels
    lab = net.labels_dev.view(-1).to(torch.int64)
    if net.lo is None:
        pos = torch.arange(1, m, device=lab.device).view(1, -1)
        side = (pos <= lab.view(-1, 1)).reshape(-1)
    else:
        lo = net.lo.to(torch.int64)
        width = (net.hi.to(torch.int64) - lo)
        site = torch.repeat_interleave(torch.arange(rows * cols, device=lab.device), width)
        start = torch.cumsum(width, 0) - width
        pos = torch.arange(int(width.sum()), device=lab.device) - start[site] + lo[site] + 1
        side = pos <= lab[site]
    term = torch.tensor([True, False], device=lab.device)
    return torch.cat([side, term]).cpu().numpy()


def extract_labeling(net: FlowNetwork, side: Optional[np.ndarray] = None) -> np.ndarray:
    """maxflow.py:362-373: per chain, lo + number of source-side chain nodes."""
    if side is None:
        if net.labels_dev is None:
            raise ValueError("network has not been solved")
        return net.labels_dev.view(net.site_shape).cpu().numpy()
    rows, cols = net.site_shape
    lo_np, hi_np = net.windows()
    lo_np, hi_np = lo_np.reshape(-1).astype(np.int64), hi_np.reshape(-1).astype(np.int64)
    width = hi_np - lo_np
    base = np.concatenate([[0], np.cumsum(width)])
    s = np.asarray(side, dtype=bool)[: base[-1]]
    counts = np.add.reduceat(s.astype(np.int64), base[:-1]) if base[-1] else np.zeros(rows * cols, np.int64)
    counts = np.where(width > 0, counts, 0)
    # a chain cut twice has a source-side node above a sink-side one
    prev = np.concatenate([[True], s[:-1]])
    first = np.zeros(base[-1], bool)
    first[base[:-1][width > 0]] = True
    bad = int(((s & ~prev) & ~first).sum())
    if bad:
        raise InternalConsistencyError(f"{bad} chains cut more than once")
    return (lo_np + counts).astype(np.int32).reshape(rows, cols)


def solve_exact(volume, params: EnergyParams, solver: str = "push-relabel", rounds_per_sweep: int = 12) -> CutResult:
    """maxflow.py:481-510: build, solve on the device, check the cut-cost identity."""
    if solver not in ("push-relabel", "dinic"):
        raise ValueError(f"unknown solver {solver!r} (push-relabel or dinic)")
    t0 = time.perf_counter()
    net = build_network(volume, params)
    build_s = time.perf_counter() - t0
    result = maxflow_push_relabel(net, rounds_per_sweep=rounds_per_sweep)
    if solver == "dinic":
        result.stats["requested_solver"] = "dinic"
    check = result.stats["labeling_energy"]
    if check != result.energy:
        raise InternalConsistencyError(f"cut cost {result.energy} != labeling energy {check}")
    result.stats.update(build_s=build_s, nodes=net.n_nodes, arcs=net.num_arcs, const_offset=net.const_offset)
    return result


def solve_exact_bands(volume, params: EnergyParams, devices=(0, 1), lo=None, hi=None) -> CutResult:
    """``solve_exact`` (maxflow.py:481-510) for one volume split into row bands,
    band k on GPU ``devices[k]`` (BASELINE config 5).

    One cooperative launch per band over that band's tile rows; the launches
    form one team, and arcs across a band edge are read and written in place
    over NVLink (gz_solve_volume_banded, include/gazecut_b200.h).  The minimum
    cut is canonical, so flow, energy and labeling are bit-identical to the
    one-GPU ``solve_exact``.  ``devices`` may repeat a GPU (its SMs are split
    between the bands it hosts).  Host arrays in, host arrays out."""
    t0 = time.perf_counter()
    vol = np.ascontiguousarray(np.asarray(volume))
    if vol.ndim != 3:
        raise ValueError("volume must be (rows, cols, num_labels)")
    if vol.size and (int(vol.min()) < 0 or int(vol.max()) > np.iinfo(np.int32).max):
        raise ValueError("data costs must be non-negative and fit the int32 device state")
    rows, cols, m = (int(s) for s in vol.shape)
    vol32 = np.ascontiguousarray(vol, dtype=np.int32)
    lo32 = hi32 = None
    if lo is not None and hi is not None:
        lo32 = np.ascontiguousarray(np.asarray(lo).reshape(rows, cols), dtype=np.int32)
        hi32 = np.ascontiguousarray(np.asarray(hi).reshape(rows, cols), dtype=np.int32)
        if (lo32 < 0).any() or (hi32 >= m).any() or (lo32 > hi32).any():
            raise ValueError("label windows must satisfy 0 <= lo <= hi < num_labels")
        if (lo32 == 0).all() and (hi32 == m - 1).all():
            lo32 = hi32 = None
    devs = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
    if devs.size < 1:
        raise ValueError("at least one band")
    _dev.require_gpu()
    labels = np.empty((rows, cols), dtype=np.int32)
    st = _lib.Stats()
    en = params._c()
    sc = _sched(12, None, True, 0)
    vp = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    rc = _lib.lib().gz_solve_volume_banded(vp(vol32), rows, cols, m, C.byref(en), C.byref(sc), vp(lo32), vp(hi32),
                                          int(devs.size), vp(devs), vp(labels), C.byref(st))
    if rc == _lib.GZ_ERR_ARG:
        raise ValueError("gz_solve_volume_banded: invalid argument (m in 2..256, one tile row per band, "
                         "valid device ids)")
    _lib.check(rc, "gz_solve_volume_banded")
    flow = int(st.flow)
    offset = int(st.const_offset)
    energy = flow + offset
    if int(st.labeling_energy) != energy:
        raise InternalConsistencyError(f"cut cost {energy} != labeling energy {int(st.labeling_energy)}")
    stats = {
        "solver": "push-relabel", "bands": int(devs.size), "devices": [int(d) for d in devs],
        "converged": bool(st.converged), "sweeps": int(st.sweeps), "pushes": int(st.pushes),
        "relabels": int(st.relabels), "presaturated": int(st.presaturated), "device": "sm_100a",
        "device_ms": float(st.ms_total), "pulses": int(st.pulses), "bfs_passes": int(st.bfs_passes),
        "reach_passes": int(st.reach_passes), "labeling_energy": int(st.labeling_energy),
        "node_updates": int(st.node_updates), "const_offset": offset, "wall_s": time.perf_counter() - t0,
        "phase_ms": {k: round(float(v), 4) for k, v in
                     zip(("init", "mask_build", "global_relabel", "pulses", "extract", "tail"), st.ms_phase)},
    }
    return CutResult(flow=flow, energy=energy, labeling=labels, stats=stats)
