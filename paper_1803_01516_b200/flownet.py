"""The cut network as an implicit device graph.

The reference materialises an Ishikawa layered graph in CSR form
(flownet.py:41-296, int32 arc ids, ~0.54 GB at 384x288x16 and over 89 GB at
1080p x 128).  Here the graph is implicit: a :class:`FlowNetwork` holds the
device-resident data volume, the energy parameters and the optional per-site
label windows; the solver kernels enumerate arcs by index arithmetic (see
csrc/gz_graph.cuh).  Graph-size bookkeeping (node/arc counts, the constant
offset of folded source->sink arcs) is evaluated on the device with closed
forms of the reference's emission rules (flownet.py:115-181).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _dev
from .energy import UNCUTTABLE, EnergyParams


def full_windows(site_shape: tuple[int, int], num_labels: int):
    """flownet.py:225-230."""
    rows, cols = site_shape
    return (np.zeros(rows * cols, np.int32), np.full(rows * cols, num_labels - 1, np.int32))


def expected_node_count(site_shape: tuple[int, int], num_labels: int) -> int:
    """sites*(m-1) + 2 (flownet.py:299-302)."""
    rows, cols = site_shape
    return rows * cols * (num_labels - 1) + 2


def expected_arc_count(site_shape: tuple[int, int], num_labels: int) -> int:
    """2*(sites*m + pairs*(m-1) + pairs*2*(m-2)) for m >= 2 (flownet.py:305-322)."""
    rows, cols = site_shape
    m = num_labels
    if m == 1:
        return 0
    sites = rows * cols
    pairs = rows * (cols - 1) + (rows - 1) * cols
    return 2 * (sites * m + pairs * (m - 1) + pairs * 2 * (m - 2))


def _span(lo, hi):
    """Length of the integer interval [lo, hi] (0 if empty), elementwise."""
    return torch.clamp(hi - lo + 1, min=0)


def _pair_counts(la, ha, lb, hb, m):
    """Per neighbour pair (a, b): emitted arc pairs and folded (source->sink)
    counts for the same-level and both diagonal families (flownet.py:146-180).
    Position t of a site is the source if t <= lo, the sink if t > hi."""
    one, top = torch.ones_like(la), torch.full_like(la, m - 1)
    ra, rb = _span(la + 1, ha), _span(lb + 1, hb)
    both = _span(torch.maximum(la, lb) + 1, torch.minimum(ha, hb))
    same = ra + rb - both
    same_off = _span(torch.maximum(one, hb + 1), torch.minimum(top, la)) + \
        _span(torch.maximum(one, ha + 1), torch.minimum(top, lb))

    def diag(lx, hx, ly, hy):   # arcs (x, t) -> (y, t-1), t in [1, m-1]
        emit = _span(torch.maximum(lx + 1, ly + 2), torch.minimum(hx, top)) + \
            _span(torch.maximum(one, ly + 2), torch.minimum(lx, hy + 1))
        off = _span(torch.maximum(one, hy + 2), torch.minimum(top, lx))
        return emit, off

    d0, o0 = diag(la, ha, lb, hb)
    d1, o1 = diag(lb, hb, la, ha)
    return same + d0 + d1, same_off, o0 + o1


def graph_size(volume: torch.Tensor, params: EnergyParams, lo: Optional[torch.Tensor],
               hi: Optional[torch.Tensor]) -> tuple[int, int, int]:
    """(n_nodes, num_arcs, const_offset) of the reference construction."""
    rows, cols, m = (int(s) for s in volume.shape)
    if lo is None:
        if m == 1:
            return 2, 0, int(volume.sum(dtype=torch.int64))
        return expected_node_count((rows, cols), m), expected_arc_count((rows, cols), m), 0
    lo2 = lo.view(rows, cols).to(torch.int64)
    hi2 = hi.view(rows, cols).to(torch.int64)
    width = hi2 - lo2
    n_nodes = int(width.sum()) + 2
    chain = torch.where(width > 0, width + 1, torch.zeros_like(width))
    collapsed = torch.gather(volume.view(rows * cols, m).to(torch.int64), 1,
                             lo2.view(-1, 1)).view(rows, cols)
    offset = int(torch.where(width == 0, collapsed, torch.zeros_like(collapsed)).sum())
    arcs = int(chain.sum())
    icap = UNCUTTABLE if params.hard_inhibit else params.inhibit
    for a_sl, b_sl in (((slice(None), slice(None, -1)), (slice(None), slice(1, None))),
                       ((slice(None, -1), slice(None)), (slice(1, None), slice(None)))):
        emit, s_off, d_off = _pair_counts(lo2[a_sl], hi2[a_sl], lo2[b_sl], hi2[b_sl], m)
        arcs += int(emit.sum())
        offset += params.penalty * int(s_off.sum()) + icap * int(d_off.sum())
    # the reference accumulates the offset in numba int64 (flownet.py:115, 124-125,
    # 153-154, 172-173), which wraps once many uncuttable (2^56) arcs fold
    offset = (offset + (1 << 63)) % (1 << 64) - (1 << 63)
    return n_nodes, 2 * arcs, offset


@dataclass
class FlowNetwork:
    """Device-resident implicit cut network (stands in for flownet.py:41-89).

    ``volume`` is the int32 CUDA data volume (rows, cols, m); ``lo``/``hi``
    the optional int32 per-site windows.  Node numbering (for
    :func:`gazecut_b200.maxflow.source_side`) follows the reference: chain
    nodes site-major (node_base = cumsum(hi - lo)), then source, then sink.
    """

    volume: torch.Tensor
    params: EnergyParams
    lo: Optional[torch.Tensor] = None
    hi: Optional[torch.Tensor] = None
    n_nodes: int = 0
    num_arcs: int = 0
    const_offset: int = 0
    # filled by a solve
    labels_dev: Optional[torch.Tensor] = field(default=None, repr=False)
    last_stats: Optional[dict] = field(default=None, repr=False)

    @property
    def site_shape(self) -> tuple[int, int]:
        return (int(self.volume.shape[0]), int(self.volume.shape[1]))

    @property
    def num_labels(self) -> int:
        return int(self.volume.shape[2])

    @property
    def source(self) -> int:
        return self.n_nodes - 2

    @property
    def sink(self) -> int:
        return self.n_nodes - 1

    @property
    def has_chains(self) -> bool:
        return True

    def windows(self):
        rows, cols = self.site_shape
        if self.lo is None:
            lo, hi = full_windows((rows, cols), self.num_labels)
            return lo.reshape(rows, cols), hi.reshape(rows, cols)
        return (self.lo.view(rows, cols).cpu().numpy(), self.hi.view(rows, cols).cpu().numpy())

    def reset(self) -> None:
        """Forget the last solution (the device state is rebuilt by every solve)."""
        self.labels_dev = None
        self.last_stats = None


def build_network(volume, params: EnergyParams, lo=None, hi=None) -> FlowNetwork:
    """flownet.py:233-296: validate windows, upload, size the graph (no CSR)."""
    vol = _dev.as_device_i32(volume, "volume")
    if vol.dim() != 3:
        raise ValueError("volume must be (rows, cols, num_labels)")
    rows, cols, m = (int(s) for s in vol.shape)
    if vol.numel() and int(vol.min()) < 0:
        raise ValueError("data costs must be non-negative")
    lo_d = hi_d = None
    if lo is not None and hi is not None:
        lo_d = _dev.as_device_i32(lo, "lo").reshape(rows * cols).contiguous()
        hi_d = _dev.as_device_i32(hi, "hi").reshape(rows * cols).contiguous()
        if bool((lo_d < 0).any()) or bool((hi_d >= m).any()) or bool((lo_d > hi_d).any()):
            raise ValueError("label windows must satisfy 0 <= lo <= hi < num_labels")
        if bool((lo_d == 0).all()) and bool((hi_d == m - 1).all()):
            lo_d = hi_d = None   # full windows: the exact construction
    n_nodes, num_arcs, offset = graph_size(vol, params, lo_d, hi_d)
    return FlowNetwork(volume=vol, params=params, lo=lo_d, hi=hi_d, n_nodes=n_nodes, num_arcs=num_arcs,
                       const_offset=offset)


def network_from_arcs(n_nodes: int, source: int, sink: int, arcs):
    """Generic CSR networks (flownet.py:325-353) are outside the B200 path.

    The device solver works on the implicit gaze-line grid only; general
    graphs are served by the reference package (scope)."""
    raise NotImplementedError("network_from_arcs: generic networks are out of scope for the B200 grid solver")
