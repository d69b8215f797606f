"""Max-flow / min-cut on the device and the cut read-out.

Mirrors ``gazecut.maxflow`` (maxflow.py:1-510).  Grid networks run the
sm_100a implicit-graph push-relabel solver (gz_solve_volume); the labeling is
the canonical minimal source side of the minimum cut, identical to the one
the reference extracts (maxflow.py:1-16), so exact solves agree bit for bit.
Explicit networks (network_from_arcs, or a grid network whose CSR arrays
were materialised) run the CSR kernel (gz_maxflow_csr) on their arrays, which
it updates in place like the reference's solvers.
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
    if nbytes == 0:
        raise ValueError(f"grid {rows}x{cols}x{m} exceeds the int32 node indexing of the device solver")
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
    if m > 1 and L.gz_workspace_bytes(rows, cols, m) and m <= 256:
        net._solved_state = (ws, _dev.workspace_generation())
    return labels, st


_PLANES = (("cu", _lib.GZ_PLANE_CHAIN), ("ph", _lib.GZ_PLANE_SAME_RIGHT), ("pv", _lib.GZ_PLANE_SAME_DOWN),
           ("dar", _lib.GZ_PLANE_DIAG_RIGHT), ("dbr", _lib.GZ_PLANE_DIAG_LEFT), ("dad", _lib.GZ_PLANE_DIAG_DOWN),
           ("dbd", _lib.GZ_PLANE_DIAG_UP), ("e", _lib.GZ_PLANE_EXCESS), ("h", _lib.GZ_PLANE_HEIGHT))


def solve_state(net: FlowNetwork, planes=("cu", "ph", "pv", "dar", "dbr", "dad", "dbd", "e")) -> dict:
    """The final device state of the last implicit-graph solve of ``net``
    (gz_export_state): int32 host arrays (sites, m-1), position t in column
    t-1 -- the residual preflow the optimality certificate checks
    (oracle/gz_certify.c).  Must be called before any other
    device call reuses the solver workspace."""
    if net._solved_state is None:
        raise ValueError("network has no implicit-solve state (solve it with maxflow_push_relabel first)")
    ws, gen = net._solved_state
    if gen != _dev.workspace_generation():
        raise RuntimeError("the solve state was overwritten by a later device call; re-solve the network")
    rows, cols = net.site_shape
    m = net.num_labels
    out = {}
    buf = torch.empty((rows * cols, m - 1), dtype=torch.int32, device=net.volume.device)
    for name, plane in _PLANES:
        if name not in planes:
            continue
        _lib.check(_lib.lib().gz_export_state(_dev.ptr(ws), rows, cols, m, plane, _dev.ptr(buf), _dev.stream_ptr()),
                   "gz_export_state")
        out[name] = buf.cpu().numpy()
    return out


# -- explicit (CSR) networks -------------------------------------------------

def _csr_device(net: FlowNetwork):
    csr = net.materialize()
    dev = _dev.require_gpu()
    def up(a):   # (a network without arcs still passes non-null arrays)
        a = np.ascontiguousarray(a)
        return torch.from_numpy(a if a.size else np.zeros(1, a.dtype)).to(dev)
    t = {k: up(csr[k]) for k in ("first_out", "head", "rev", "cap", "resid")}
    return csr, t


def _csr_solve(net: FlowNetwork, rounds_per_sweep: int, max_sweeps: Optional[int], want_side: bool = True):
    """gz_maxflow_csr on the network's arrays; resid is written back in place."""
    csr, t = _csr_device(net)
    n = net.n_nodes
    L = _lib.lib()
    nbytes = L.gz_csr_workspace_bytes(n)
    ws = _dev.csr_workspace(nbytes)
    side = torch.empty(n, dtype=torch.uint8, device=t["cap"].device) if want_side else None
    st = _lib.CsrStats()
    rc = L.gz_maxflow_csr(n, net.source, net.sink, _dev.ptr(t["first_out"]), _dev.ptr(t["head"]),
                          _dev.ptr(t["rev"]), _dev.ptr(t["cap"]), _dev.ptr(t["resid"]), int(rounds_per_sweep),
                          -1 if max_sweeps is None else int(max_sweeps),
                          _dev.ptr(side) if side is not None else None, None, C.byref(st), _dev.ptr(ws), nbytes,
                          _dev.stream_ptr())
    _lib.check(rc, "gz_maxflow_csr")
    csr["resid"][:] = t["resid"].cpu().numpy()[: csr["resid"].size]
    return st, (side.cpu().numpy().astype(bool) if side is not None else None)


def chain_presaturate(net: FlowNetwork) -> int:
    """maxflow.py:341-352: push each chain's minimum residual straight through it
    (on the device, on the network's CSR arrays); returns the amount pushed."""
    if not net.has_chains:
        return 0
    csr, t = _csr_device(net)
    dev = t["cap"].device
    ca = torch.from_numpy(np.ascontiguousarray(csr["chain_arcs"])).to(dev)
    cb = torch.from_numpy(np.ascontiguousarray(csr["chain_base"])).to(dev)
    sent = torch.zeros(1, dtype=torch.int64, device=dev)
    nsites = int(csr["chain_base"].size - 1)
    _lib.check(_lib.lib().gz_chain_presaturate_csr(_dev.ptr(t["rev"]), _dev.ptr(t["resid"]), _dev.ptr(ca),
                                                   _dev.ptr(cb), nsites, _dev.ptr(sent), _dev.stream_ptr()),
               "gz_chain_presaturate_csr")
    csr["resid"][:] = t["resid"].cpu().numpy()[: csr["resid"].size]
    return int(sent.item())


def conservation_violations(net: FlowNetwork) -> int:
    """maxflow.py:376-382: non-terminal nodes whose net flow is not zero (device)."""
    resid = net.resid            # (a solved grid network's state first becomes a flow)
    csr, t = _csr_device(net)
    if resid.size:
        t["resid"] = torch.from_numpy(np.ascontiguousarray(resid)).to(t["cap"].device)
    bad = torch.zeros(1, dtype=torch.int64, device=t["cap"].device)
    _lib.check(_lib.lib().gz_conservation_violations_csr(_dev.ptr(t["first_out"]), _dev.ptr(t["cap"]),
                                                         _dev.ptr(t["resid"]), net.n_nodes, net.source, net.sink,
                                                         _dev.ptr(bad), _dev.stream_ptr()),
               "gz_conservation_violations_csr")
    return int(bad.item())


def _csr_result(net: FlowNetwork, st, side, solver: str, t0: float, presat: int) -> CutResult:
    converged = bool(st.converged)
    stats = {
        "solver": solver,
        "wall_s": time.perf_counter() - t0,
        "converged": converged,
        "sweeps": int(st.sweeps),
        "pushes": int(st.pushes),
        "relabels": int(st.relabels),
        "presaturated": presat,
        "stranded_excess_nodes": int(st.stranded_excess_nodes),
        "device": "sm_100a",
        "device_ms": float(st.ms_total),
        "pulses": int(st.pulses),
        "engine": "gz_maxflow_csr (push-relabel with global relabeling on the explicit CSR network)",
    }
    net.last_stats = stats
    result = CutResult(flow=int(st.flow), source_side=side, stats=stats)
    if net.has_chains:
        result.labeling = extract_labeling(net, side)
        net.labels_dev = torch.from_numpy(result.labeling.reshape(-1).astype(np.int32)).to(net.volume.device)
        if converged:
            result.energy = result.flow + net.const_offset
    return result


def maxflow_push_relabel(net: FlowNetwork, rounds_per_sweep: int = 12, max_sweeps: Optional[int] = None,
                         block: Optional[int] = None, presaturate: bool = True) -> CutResult:
    """Preflow-push with global relabeling on the device (maxflow.py:403-478).

    Grid networks: the implicit-graph kernel.  ``max_sweeps`` caps the number
    of sweeps (global relabel + pulses): the level-2 approximation,
    ``stats['converged']`` False when the cap bit.  ``block`` is accepted for
    API parity; the device's capped schedule is its own deterministic one
    (DESIGN.md §2).  Explicit networks (generic, or grid networks whose CSR
    arrays were materialised): the CSR kernel on ``net.resid`` in place."""
    if rounds_per_sweep < 1:
        raise ValueError("rounds_per_sweep must be >= 1")
    t0 = time.perf_counter()
    if not net.is_grid or net.materialized:
        presat = chain_presaturate(net) if presaturate and net.has_chains else 0
        st, side = _csr_solve(net, rounds_per_sweep, max_sweeps)
        return _csr_result(net, st, side, "push-relabel", t0, presat)
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
    flow = int(st.flow)
    stats["flow"] = flow
    net.last_stats = stats
    result = CutResult(flow=flow, stats=stats)
    result.labeling = labels.view(net.site_shape).cpu().numpy()
    result.source_side = source_side(net)
    if converged:
        result.energy = flow + net.const_offset
    return result


def maxflow_reference(net: FlowNetwork) -> CutResult:
    """maxflow.py:385-400, the reference's second exact solver (Dinic there).

    Here it is the OTHER device engine: the network is materialised from the
    device graph and solved by the explicit-CSR kernel (gz_maxflow_csr),
    independent of the implicit-graph kernel ``maxflow_push_relabel`` runs on
    grid networks.  The minimum cut is canonical, so flow and labeling agree
    with Dinic's; ``stats['solver']`` is "dinic" (the contract of
    pkg/tests/test_maxflow.py:154) and ``stats['engine']`` says what ran."""
    t0 = time.perf_counter()
    st, side = _csr_solve(net, 12, None)
    r = _csr_result(net, st, side, "dinic", t0, 0)
    r.stats["converged"] = True
    return r


def source_side(net: FlowNetwork) -> np.ndarray:
    """maxflow.py:355-359: bool per node (chains site-major, source, sink).

    Grid networks solved by the implicit kernel: chains are cut exactly once
    (uncuttable reverse arcs), so the source side of site s is chain positions
    lo+1 .. label, derived on the device from the labels.  Explicit networks:
    BFS from the source over resid > 0 on the device (gz_source_side_csr)."""
    if not net.is_grid or net.materialized:
        csr, t = _csr_device(net)
        side = torch.empty(net.n_nodes, dtype=torch.uint8, device=t["cap"].device)
        _lib.check(_lib.lib().gz_source_side_csr(net.n_nodes, net.source, _dev.ptr(t["first_out"]),
                                                 _dev.ptr(t["head"]), _dev.ptr(t["resid"]), _dev.ptr(side),
                                                 _dev.stream_ptr()), "gz_source_side_csr")
        return side.cpu().numpy().astype(bool)
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
    if not net.has_chains:
        raise ValueError("network has no chain metadata")
    if side is None:
        if net.is_grid and not net.materialized and net.labels_dev is not None:
            return net.labels_dev.view(net.site_shape).cpu().numpy()
        side = source_side(net)
    rows, cols = net.site_shape
    lo_np, hi_np = net.windows()
    lo_np, hi_np = lo_np.reshape(-1).astype(np.int64), hi_np.reshape(-1).astype(np.int64)
    width = hi_np - lo_np
    base = np.concatenate([[0], np.cumsum(width)])
    s = np.asarray(side, dtype=bool)[: base[-1]]
    cs = np.concatenate([[0], np.cumsum(s, dtype=np.int64)])
    counts = cs[base[1:]] - cs[base[:-1]]
    # a chain cut twice has a source-side node above a sink-side one
    prev = np.concatenate([[True], s[:-1]])
    first = np.zeros(base[-1], bool)
    first[base[:-1][width > 0]] = True
    bad = int(((s & ~prev) & ~first).sum())
    if bad:
        raise InternalConsistencyError(f"{bad} chains cut more than once")
    return (lo_np + counts).astype(np.int32).reshape(rows, cols)


def solve_exact(volume, params: EnergyParams, solver: str = "push-relabel", rounds_per_sweep: int = 12) -> CutResult:
    """maxflow.py:481-510: build, solve on the device, check the cut-cost identity.

    ``solver="push-relabel"``: the implicit-graph kernel; ``"dinic"``: the
    reference's second solver slot, here the explicit-CSR device kernel on the
    materialised graph (:func:`maxflow_reference`)."""
    if solver not in ("push-relabel", "dinic"):
        raise ValueError(f"unknown solver {solver!r} (push-relabel or dinic)")
    t0 = time.perf_counter()
    net = build_network(volume, params)
    build_s = time.perf_counter() - t0
    if solver == "push-relabel":
        result = maxflow_push_relabel(net, rounds_per_sweep=rounds_per_sweep)
        check = result.stats["labeling_energy"]
    else:
        result = maxflow_reference(net)
        from .energy import total_energy_device
        check = total_energy_device(net.labels_dev, net.volume, params)
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
