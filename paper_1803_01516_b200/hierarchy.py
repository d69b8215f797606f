"""Hierarchical approximation on the device (hierarchy.py:1-165).

Level 1: coarsen by ``b`` in all three axes (gz_coarsen), cut the coarse
volume exactly, derive per-site windows around the upsampled coarse surface
(gz_thin_skin), cut the fine volume exactly inside them.  Level 2: same
skin, but the fine cut stops after ``max_sweeps`` sweeps.  Everything stays
on the GPU between the stages.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import replace
from typing import Optional

import numpy as np
import torch

from . import _dev, _lib
from .energy import EnergyParams, total_energy_device
from .flownet import build_network
from .maxflow import CutResult, InternalConsistencyError, maxflow_push_relabel

DEFAULT_SKIN_RADIUS = 1   # hierarchy.py:35
DEFAULT_L2_SWEEPS = 8     # hierarchy.py:36


def coarsen_device(vol: torch.Tensor, block: int) -> torch.Tensor:
    rows, cols, m = (int(s) for s in vol.shape)
    rb, cb, mb = -(-rows // block), -(-cols // block), -(-m // block)
    out = torch.empty((rb, cb, mb), dtype=torch.int32, device=vol.device)
    _lib.check(_lib.lib().gz_coarsen(_dev.ptr(vol), rows, cols, m, block, _dev.ptr(out), _dev.stream_ptr()),
               "gz_coarsen")
    return out


def coarsen(volume, block: int, params: EnergyParams):
    """hierarchy.py:39-57: zero-padded b^3 sums, penalty * b."""
    if block < 1:
        raise ValueError("block must be >= 1")
    vol = _dev.as_device_i32(volume, "volume")
    if int(vol.sum(dtype=torch.int64)) > _dev.INT32_MAX:
        raise ValueError("coarse volume exceeds the int32 device representation")
    return coarsen_device(vol, block).cpu().numpy().astype(np.int64), replace(params, penalty=params.penalty * block)


def thin_skin_device(coarse_lab: torch.Tensor, fine_shape, block: int, radius: int):
    rows, cols, m = fine_shape
    lo = torch.empty(rows * cols, dtype=torch.int32, device=coarse_lab.device)
    hi = torch.empty_like(lo)
    crows, ccols = (int(s) for s in coarse_lab.shape)
    _lib.check(_lib.lib().gz_thin_skin(_dev.ptr(coarse_lab), crows, ccols, rows, cols, m, block, radius,
                                       _dev.ptr(lo), _dev.ptr(hi), _dev.stream_ptr()), "gz_thin_skin")
    return lo, hi


def thin_skin(coarse_labeling, fine_shape, block: int, radius: int = DEFAULT_SKIN_RADIUS):
    """hierarchy.py:60-73: windows [b(D-r), b(D+r+1)-1] clamped to [0, m-1]."""
    lab = _dev.as_device_i32(coarse_labeling, "coarse_labeling")
    rows, cols, _ = fine_shape
    if lab.dim() != 2 or int(lab.shape[0]) * block < rows or int(lab.shape[1]) * block < cols:
        raise ValueError(f"coarse labeling {tuple(lab.shape)} x block {block} does not cover the fine grid "
                         f"{(rows, cols)}")
    lo, hi = thin_skin_device(lab, fine_shape, block, radius)
    return lo.view(rows, cols).cpu().numpy(), hi.view(rows, cols).cpu().numpy()


def _exact(vol: torch.Tensor, params: EnergyParams, lo, hi, rounds_per_sweep: int,
           solver: str = "push-relabel") -> tuple[CutResult, object]:
    """hierarchy.py:76-89 _solve_restricted_exact: windowed build, exact solve,
    cut-cost identity.  ``solver="dinic"`` runs the explicit-CSR device kernel
    (maxflow.maxflow_reference) instead of the implicit-graph one."""
    net = build_network(vol, params, lo=lo, hi=hi)
    if solver == "dinic":
        from .energy import total_energy_device
        from .maxflow import maxflow_reference
        result = maxflow_reference(net)
        result.stats["labeling_energy"] = total_energy_device(net.labels_dev, net.volume, params)
    else:
        result = maxflow_push_relabel(net, rounds_per_sweep=rounds_per_sweep)
    if result.stats["labeling_energy"] != result.energy:
        raise InternalConsistencyError(
            f"cut cost {result.energy} != labeling energy {result.stats['labeling_energy']}")
    result.stats["nodes"] = net.n_nodes
    result.stats["arcs"] = net.num_arcs
    return result, net


def _coarse_stage(volume, params, block, skin_radius, rounds_per_sweep):
    vol = _dev.as_device_i32(volume, "volume")
    if block < 1:
        raise ValueError("block must be >= 1")
    if int(vol.sum(dtype=torch.int64)) > _dev.INT32_MAX:
        raise ValueError("coarse volume exceeds the int32 device representation")
    cvol = coarsen_device(vol, block)
    cparams = replace(params, penalty=params.penalty * block)
    coarse, cnet = _exact(cvol, cparams, None, None, rounds_per_sweep)
    lo, hi = thin_skin_device(cnet.labels_dev.view(cvol.shape[0], cvol.shape[1]), tuple(vol.shape), block,
                              skin_radius)
    return vol, coarse, lo, hi


def solve_level1(volume, params: EnergyParams, block: int, skin_radius: int = DEFAULT_SKIN_RADIUS,
                 solver: str = "push-relabel", rounds_per_sweep: int = 12) -> CutResult:
    """hierarchy.py:92-117."""
    t0 = time.perf_counter()
    if solver not in ("push-relabel", "dinic"):
        raise ValueError(f"unknown solver {solver!r} (push-relabel or dinic)")
    vol, coarse, lo, hi = _coarse_stage(volume, params, block, skin_radius, rounds_per_sweep)
    result, _ = _exact(vol, params, lo, hi, rounds_per_sweep, solver)
    result.stats.update(
        level=1, block=block, skin_radius=skin_radius, coarse_energy=coarse.energy,
        coarse_wall_s=coarse.stats["wall_s"], mean_window=float((hi - lo + 1).double().mean()),
        coarse_device_ms=coarse.stats["device_ms"],
        device_ms_total=coarse.stats["device_ms"] + result.stats["device_ms"], wall_s=time.perf_counter() - t0)
    return result


def solve_level2(volume, params: EnergyParams, block: int, skin_radius: int = DEFAULT_SKIN_RADIUS,
                 rounds_per_sweep: int = 12, max_sweeps: Optional[int] = DEFAULT_L2_SWEEPS) -> CutResult:
    """hierarchy.py:120-165: capped fine solve inside the skin; energy recomputed
    from the labeling.  ``max_sweeps=None`` makes it identical to level 1."""
    t0 = time.perf_counter()
    vol, coarse, lo, hi = _coarse_stage(volume, params, block, skin_radius, rounds_per_sweep)
    net = build_network(vol, params, lo=lo, hi=hi)
    result = maxflow_push_relabel(net, rounds_per_sweep=rounds_per_sweep, max_sweeps=max_sweeps, block=block)
    result.energy = int(result.stats["labeling_energy"])
    if result.stats["converged"] and result.energy != result.flow + net.const_offset:
        raise InternalConsistencyError(
            f"cut cost {result.flow + net.const_offset} != labeling energy {result.energy}")
    result.stats.update(
        level=2, block=block, skin_radius=skin_radius, coarse_energy=coarse.energy,
        coarse_wall_s=coarse.stats["wall_s"], mean_window=float((hi - lo + 1).double().mean()),
        coarse_device_ms=coarse.stats["device_ms"],
        device_ms_total=coarse.stats["device_ms"] + result.stats["device_ms"],
        nodes=net.n_nodes, arcs=net.num_arcs, wall_s=time.perf_counter() - t0)
    return result
