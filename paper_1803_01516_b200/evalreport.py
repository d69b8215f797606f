"""Accuracy accounting and penalty sweeps on the device (evalreport.py:1-126
of the reference).

``error_count`` runs gz_error_count; ``sweep_penalty`` solves every penalty of
the sweep with gz_solve_volume_batch (up to 8 exact solves in flight) and
counts errors on the device, so no labeling makes a host round trip.
``compare_methods`` and the CSV writers are the reference's reporting
callers, kept so experiment scripts switch over unchanged."""

from __future__ import annotations

import csv
import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _dev, _lib
from .energy import EnergyParams
from .imaging import GroundTruthDepth

HISTOGRAM_TAIL = 9  # |error| >= this shares the last bucket (evalreport.py:18)


@dataclass
class ErrorReport:
    """evalreport.py:21-44."""

    total_error: int
    evaluated: int
    histogram: np.ndarray
    tail: int = HISTOGRAM_TAIL

    @property
    def exact_fraction(self) -> float:
        return float(self.histogram[0] / self.evaluated) if self.evaluated else 0.0

    def rows(self):
        out = [(str(k), int(self.histogram[k])) for k in range(self.tail)]
        out.append((f"{self.tail}~", int(self.histogram[self.tail])))
        return out


def _reports(out: torch.Tensor, tail: int) -> list[ErrorReport]:
    o = out.cpu().numpy().reshape(-1, tail + 3)
    return [ErrorReport(total_error=int(r[0]), evaluated=int(r[1]), histogram=r[2:].astype(np.int64), tail=tail)
            for r in o]


def error_count_device(labels: torch.Tensor, gt: GroundTruthDepth, tail: int = HISTOGRAM_TAIL) -> list[ErrorReport]:
    """error_count for a batch of device labelings (batch, rows, cols)."""
    depth, valid = gt.device_arrays()
    lab = labels.to(depth.device, dtype=torch.int32).contiguous()
    rows, cols = depth.shape
    batch = lab.numel() // (rows * cols)
    if lab.numel() != batch * rows * cols or batch < 1:
        raise ValueError(f"labeling shape {tuple(labels.shape)} != ground truth {tuple(depth.shape)}")
    out = torch.empty(batch * (tail + 3), dtype=torch.int64, device=depth.device)
    rc = _lib.lib().gz_error_count(_dev.ptr(lab), batch, _dev.ptr(depth), _dev.ptr(valid), rows, cols, int(tail),
                                   _dev.ptr(out), _dev.stream_ptr())
    _lib.check(rc, "gz_error_count")
    return _reports(out, tail)


def error_count(labeling, gt: GroundTruthDepth, tail: int = HISTOGRAM_TAIL) -> ErrorReport:
    """evalreport.py:47-61: sum of |label - depth| over ground-truth sites."""
    shape = tuple(labeling.shape) if hasattr(labeling, "shape") else np.asarray(labeling).shape
    if shape != tuple(np.asarray(gt.depth).shape):
        raise ValueError(f"labeling shape {shape} != ground truth {np.asarray(gt.depth).shape}")
    lab = _dev.as_device_i32(labeling, "labeling")
    return error_count_device(lab.unsqueeze(0), gt, tail)[0]


def error_from_histogram(histogram) -> int:
    """evalreport.py:64-76 (host arithmetic on a ten-entry histogram)."""
    items = histogram.items() if isinstance(histogram, dict) else enumerate(histogram)
    return int(sum(int(k) * int(c) for k, c in items))


@dataclass
class SweepRecord:
    """evalreport.py:79-86."""

    penalty: int
    energy: int
    flow: int
    error: int
    exact_fraction: float
    wall_s: float = 0.0


def sweep_penalty(volume, gt: GroundTruthDepth, penalties: Sequence[int], inhibit: int = 1023,
                  hard_inhibit: bool = False, solver: str = "push-relabel", progress=None) -> list[SweepRecord]:
    """evalreport.py:88-126: an exact solve per penalty, one record each.

    All penalties go to the device in one gz_solve_volume_batch call (up to 8
    solves in flight); labelings stay on the device for gz_error_count.
    ``wall_s`` is the batch's wall time divided evenly over the records."""
    if solver not in ("push-relabel", "dinic"):
        raise ValueError(f"unknown solver {solver!r} (push-relabel or dinic)")
    pens = [int(p) for p in penalties]
    if not pens:
        return []
    t0 = time.perf_counter()
    vol = _dev.as_device_i32(volume, "volume")
    if vol.dim() != 3:
        raise ValueError("volume must be (rows, cols, num_labels)")
    if vol.numel() and int(vol.min()) < 0:
        raise ValueError("data costs must be non-negative")
    rows, cols, m = (int(s) for s in vol.shape)
    n = len(pens)
    energies = (_lib.Energy * n)(*[EnergyParams(p, inhibit, hard_inhibit)._c() for p in pens])
    stats = (_lib.Stats * n)()
    labels = torch.empty((n, rows, cols), dtype=torch.int32, device=vol.device)
    if m < 2:   # single label: every site takes label 0 (flownet.py:305-322)
        from .energy import total_energy
        e = total_energy(np.zeros((rows, cols), np.int32), volume, EnergyParams(pens[0], inhibit, hard_inhibit))
        labels.zero_()
        for i in range(n):
            stats[i].energy = stats[i].labeling_energy = stats[i].const_offset = e
    else:
        L = _lib.lib()
        one = L.gz_workspace_bytes(rows, cols, m)
        ws = _dev.workspace(one * min(8, n) + 4096)
        sc = _lib.Sched(12, 0, 0, 0)
        rc = L.gz_solve_volume_batch(_dev.ptr(vol), rows, cols, m, energies, n, C.byref(sc), _dev.ptr(labels),
                                     stats, _dev.ptr(ws), ws.numel(), _dev.stream_ptr())
        if rc == _lib.GZ_ERR_CONSISTENCY:
            from .maxflow import InternalConsistencyError
            raise InternalConsistencyError("cut cost != labeling energy in a penalty sweep solve")
        _lib.check(rc, "gz_solve_volume_batch")
    reports = error_count_device(labels, gt)
    wall = (time.perf_counter() - t0) / n
    records = []
    for i, p in enumerate(pens):
        st = stats[i]
        energy = int(st.energy)
        flow = int(st.flow) if m >= 2 else 0
        records.append(SweepRecord(penalty=p, energy=energy, flow=flow, error=reports[i].total_error,
                                   exact_fraction=reports[i].exact_fraction, wall_s=wall))
        if progress:
            print(f"penalty {p:3d}: error {reports[i].total_error} exact {reports[i].exact_fraction:.1%}",
                  file=progress)
    return records


def best_penalty(records: Sequence[SweepRecord]) -> int:
    """evalreport.py:129-132: penalty of the smallest error (first on ties)."""
    return min(records, key=lambda r: (r.error, r.penalty)).penalty


@dataclass
class MethodRow:
    """evalreport.py:135-145: one (level, block) configuration's outcome."""

    level: int
    block: int
    energy: int
    error: Optional[int]
    exact_fraction: Optional[float]
    wall_s: float
    nodes: int
    converged: bool = True


def compare_methods(volume, params: EnergyParams, configs: Sequence[tuple[int, int]],
                    gt: Optional[GroundTruthDepth] = None, skin_radius: int = 1, max_sweeps: Optional[int] = None,
                    progress=None) -> list[MethodRow]:
    """evalreport.py:148-186: run (level, block) configurations on one volume
    (level 0 exact, 1 and 2 the hierarchy); errors counted on the device."""
    from .hierarchy import solve_level1, solve_level2
    from .maxflow import solve_exact
    vol = _dev.as_device_i32(volume, "volume")
    out = []
    for level, block in configs:
        if level not in (0, 1, 2):
            raise ValueError(f"unknown level {level} (0, 1 or 2)")
        t0 = time.perf_counter()
        if level == 0:
            res = solve_exact(vol, params)
        elif level == 1:
            res = solve_level1(vol, params, block, skin_radius=skin_radius)
        else:
            extra = {} if max_sweeps is None else {"max_sweeps": max_sweeps}
            res = solve_level2(vol, params, block, skin_radius=skin_radius, **extra)
        wall = time.perf_counter() - t0
        rep = error_count(res.labeling, gt) if gt is not None else None
        out.append(MethodRow(level=level, block=block, energy=res.energy,
                             error=None if rep is None else rep.total_error,
                             exact_fraction=None if rep is None else rep.exact_fraction, wall_s=wall,
                             nodes=int(res.stats.get("nodes", 0)), converged=bool(res.stats.get("converged", True))))
        if progress:
            tail = "" if rep is None else f" error {rep.total_error}"
            print(f"level {level} block {block}: energy {res.energy}{tail}", file=progress)
    return out


def _csv_target(path_or_file):
    """(stream, close?) for a path or an already open text stream."""
    if hasattr(path_or_file, "write"):
        return path_or_file, False
    return open(path_or_file, "w", newline=""), True


def _write_csv(path_or_file, comments, header, rows) -> None:
    f, close = _csv_target(path_or_file)
    try:
        for c in comments:
            f.write(f"# {c}\n")
        w = csv.writer(f)
        w.writerow(header)
        w.writerows(rows)
    finally:
        if close:
            f.close()


def write_sweep_csv(path, records: Sequence[SweepRecord], comments=(), timings=False) -> None:
    """evalreport.py:197-210: penalty,energy,flow,error,exact_fraction[,wall_s]."""
    header = ["penalty", "energy", "flow", "error", "exact_fraction"] + (["wall_s"] if timings else [])
    rows = [[r.penalty, r.energy, r.flow, r.error, f"{r.exact_fraction:.6f}"] + ([f"{r.wall_s:.3f}"] if timings else [])
            for r in records]
    _write_csv(path, comments, header, rows)


def write_compare_csv(path, rows: Sequence[MethodRow], comments=(), timings=False) -> None:
    """evalreport.py:213-233: level,block,energy,error,exact_fraction,nodes,converged[,wall_s]."""
    header = ["level", "block", "energy", "error", "exact_fraction", "nodes", "converged"] + \
        (["wall_s"] if timings else [])
    body = [[r.level, r.block, r.energy, "" if r.error is None else r.error,
             "" if r.exact_fraction is None else f"{r.exact_fraction:.6f}", r.nodes, int(r.converged)] +
            ([f"{r.wall_s:.3f}"] if timings else []) for r in rows]
    _write_csv(path, comments, header, body)
