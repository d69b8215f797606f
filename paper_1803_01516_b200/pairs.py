"""Fused stereo-pair solving: data term + exact cut per pair in one C-ABI call.

This is the path ``bench.py`` measures: ``sad_volume`` (energy.py:83-114)
followed by ``solve_exact`` (maxflow.py:481-510) for a batch of pairs,
without materialising the int64 volume on the host.  ``solve_host`` is the
reference-facing end-to-end call (host buffers in, host labels out).
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Sequence
from typing import Optional

import numpy as np
import torch

from . import _dev, _lib
from .energy import EnergyParams, cuboid_struct
from .geometry import CuboidSpec
from .maxflow import CutResult, InternalConsistencyError


def _stats_dict(st: _lib.Stats) -> dict:
    return {
        "flow": int(st.flow), "energy": int(st.energy),
        "solver": "push-relabel", "converged": bool(st.converged), "sweeps": int(st.sweeps),
        "pushes": int(st.pushes), "relabels": int(st.relabels), "presaturated": int(st.presaturated),
        "stranded_excess_nodes": int(st.stranded_excess_nodes), "pulses": int(st.pulses),
        "bfs_passes": int(st.bfs_passes), "reach_passes": int(st.reach_passes),
        "device_ms": float(st.ms_total), "labeling_energy": int(st.labeling_energy),
        "node_updates": int(st.node_updates),
        "phase_ms": {k: round(float(v), 4) for k, v in
                     zip(("init", "mask_build", "global_relabel", "pulses", "extract", "tail"), st.ms_phase)},
    }


class PairStats(Sequence):
    """Per-pair stats of one batched call: a read-only sequence of dicts over the
    C ABI's stats array (already in host memory when the call returns); each
    pair's dict is built on first access, so a large batch does not pay for
    Python objects nobody reads."""

    def __init__(self, arr):
        self._arr = arr
        self._cache = {}

    def __len__(self) -> int:
        return len(self._arr)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        n = len(self._arr)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("pair index out of range")
        d = self._cache.get(i)
        if d is None:
            d = self._cache[i] = _stats_dict(self._arr[i])
        return d


class PairSolver:
    """Reusable device workspace for solving pairs of one image/cuboid shape."""

    def __init__(self, cuboid: CuboidSpec, params: EnergyParams, height: int, width: int, channels: int = 3,
                 rounds_per_sweep: int = 12, bfs_cap: int = 0):
        self.dev = _dev.require_gpu()
        cuboid.check_consistent(width, height)
        if cuboid.num_labels < 2:
            raise ValueError("pair solving needs at least two labels")
        self.cuboid, self.params = cuboid, params
        self.h, self.w, self.ch = height, width, channels
        self.cs = cuboid_struct(cuboid, width)
        self.cs.height = height
        self.en = params._c()
        self.sc = _lib.Sched(int(rounds_per_sweep), 0, int(bfs_cap), 0)
        self.sites = cuboid.y_extent * cuboid.g_extent
        self.ws_one = _lib.lib().gz_workspace_bytes(cuboid.y_extent, cuboid.g_extent, cuboid.num_labels)
        self._ws: Optional[torch.Tensor] = None

    def _workspace(self, extra: int = 0, batch: int = 1) -> torch.Tensor:
        # room for every pair solve the device keeps in flight (one workspace
        # slice per team of the batched launch; gz_pairs_workspace_bytes)
        y, g, m = self.cuboid.y_extent, self.cuboid.g_extent, self.cuboid.num_labels
        need = max(self.ws_one, _lib.lib().gz_pairs_workspace_bytes(y, g, m, max(1, batch))) + extra + 4096
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.dev)
        return self._ws

    def launches(self, batch: int) -> int:
        """Kernel launches one ``solve`` of ``batch`` pairs makes (1, or 2 with the
        batched tail launch; -1: the per-pair launch path)."""
        y, g, m = self.cuboid.y_extent, self.cuboid.g_extent, self.cuboid.num_labels
        n = _lib.lib().gz_pairs_launches(y, g, m, int(batch), self._workspace(0, batch).numel())
        if n < -1:
            _lib.check(n, "gz_pairs_launches")
        return n

    def solve(self, left: torch.Tensor, right: torch.Tensor, labels: Optional[torch.Tensor] = None):
        """Device batch (B, h, w, ch) uint8 -> labels (B, y_extent, g_extent) int32 + per-pair stats."""
        if left.dim() == 3:
            left, right = left.unsqueeze(0), right.unsqueeze(0)
        b = int(left.shape[0])
        if tuple(left.shape[1:]) != (self.h, self.w, self.ch) or left.shape != right.shape:
            raise ValueError("pair batch shape does not match the solver")
        if left.device != self.dev or left.dtype != torch.uint8 or not left.is_contiguous():
            left = left.to(self.dev, torch.uint8).contiguous()
        if right.device != self.dev or right.dtype != torch.uint8 or not right.is_contiguous():
            right = right.to(self.dev, torch.uint8).contiguous()
        if labels is None:
            labels = torch.empty((b, self.cuboid.y_extent, self.cuboid.g_extent), dtype=torch.int32, device=self.dev)
        stats = (_lib.Stats * b)()
        ws = self._workspace(0, b)
        rc = _lib.lib().gz_solve_pairs(_dev.ptr(left), _dev.ptr(right), b, self.h, self.w, self.ch,
                                       C.byref(self.cs), C.byref(self.en), C.byref(self.sc), _dev.ptr(labels),
                                       stats, _dev.ptr(ws), ws.numel(), _dev.stream_ptr())
        if rc == _lib.GZ_ERR_CONSISTENCY:
            raise InternalConsistencyError("cut cost != labeling energy")
        _lib.check(rc, "gz_solve_pairs")
        return labels, PairStats(stats)

    def solve_host(self, left: np.ndarray, right: np.ndarray, labels: Optional[np.ndarray] = None):
        """Host batch in, host labels out (H2D + solve + D2H in one C-ABI call)."""
        left = np.ascontiguousarray(left, dtype=np.uint8)
        right = np.ascontiguousarray(right, dtype=np.uint8)
        if left.ndim == 3:
            left, right = left[None], right[None]
        b = left.shape[0]
        if labels is None:
            labels = np.empty((b, self.cuboid.y_extent, self.cuboid.g_extent), np.int32)
        img = left[0].nbytes
        extra = 2 * (b * img + 256) + b * self.sites * 4 + 256
        ws = self._workspace(extra, b)
        stats = (_lib.Stats * b)()
        rc = _lib.lib().gz_solve_pairs_host(
            left.ctypes.data_as(C.c_void_p), right.ctypes.data_as(C.c_void_p), b, self.h, self.w, self.ch,
            C.byref(self.cs), C.byref(self.en), C.byref(self.sc), labels.ctypes.data_as(C.c_void_p), stats,
            _dev.ptr(ws), ws.numel(), _dev.stream_ptr())
        if rc == _lib.GZ_ERR_CONSISTENCY:
            raise InternalConsistencyError("cut cost != labeling energy")
        _lib.check(rc, "gz_solve_pairs_host")
        return labels, PairStats(stats)


def solve_pairs(left, right, cuboid: CuboidSpec, params: EnergyParams, rounds_per_sweep: int = 12) -> list[CutResult]:
    """Batch version of ``solve_exact(sad_volume(left, right, cuboid), params)``."""
    arr = left if isinstance(left, torch.Tensor) else np.asarray(left)
    if arr.ndim == 3:
        h, w, ch = arr.shape
    else:
        _, h, w, ch = arr.shape
    solver = PairSolver(cuboid, params, h, w, ch, rounds_per_sweep)
    labels, stats = solver.solve(torch.as_tensor(np.asarray(left)) if not isinstance(left, torch.Tensor) else left,
                                 torch.as_tensor(np.asarray(right)) if not isinstance(right, torch.Tensor) else right)
    out = []
    for i, st in enumerate(stats):
        st["const_offset"] = 0
        out.append(CutResult(flow=int(st["flow"]), energy=int(st["energy"]),
                             labeling=labels[i].cpu().numpy(), stats=st))
    return out
