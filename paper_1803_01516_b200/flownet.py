"""The cut network: an implicit device graph, materialised on demand.

The reference materialises an Ishikawa layered graph in CSR form
(flownet.py:41-296, int32 arc ids, ~0.54 GB at 384x288x16 and over 89 GB at
1080p x 128).  Here the graph is implicit: a :class:`FlowNetwork` built by
:func:`build_network` holds the device-resident data volume, the energy
parameters and the optional per-site label windows; the solver kernels
enumerate arcs by index arithmetic (csrc/gz_graph.cuh).  Graph-size
bookkeeping uses closed forms of the reference's emission rules
(flownet.py:115-181).

The reference's CSR arrays (``first_out``, ``head``, ``rev``, ``cap``,
``resid``, ``node_base``, ``chain_arcs``, ``chain_base``) are available on
every network: touching one materialises the DEVICE graph -- the solver's own
initialisation exports its arc pairs in ``_emit`` order (gz_export_arcs) and
:func:`pairs_to_csr` lays them out exactly as flownet.py:184-222 does.  Generic
networks (:func:`network_from_arcs`) are explicit from the start and are
solved by the CSR kernel (gz_maxflow_csr).
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


def pairs_to_csr(n_nodes: int, pu, pv, pc, prc):
    """flownet.py:184-222 _pairs_to_csr: arc pair i puts its forward arc in u's
    out-list and its reverse arc in v's, lists in pair order.  Returns
    (first_out int64, head int32, rev int32, cap int64, pair_arc int64)."""
    pu, pv = np.asarray(pu, np.int64), np.asarray(pv, np.int64)
    npairs = pu.size
    tails = np.empty(2 * npairs, np.int64)
    tails[0::2], tails[1::2] = pu, pv            # event 2i: forward arc, 2i+1: reverse arc
    order = np.argsort(tails, kind="stable")     # CSR position -> event
    pos = np.empty(2 * npairs, np.int64)
    pos[order] = np.arange(2 * npairs)           # event -> CSR position
    first_out = np.zeros(n_nodes + 1, np.int64)
    np.cumsum(np.bincount(tails, minlength=n_nodes), out=first_out[1:])
    head = np.empty(2 * npairs, np.int32)
    rev = np.empty(2 * npairs, np.int32)
    cap = np.empty(2 * npairs, np.int64)
    fw, bw = pos[0::2], pos[1::2]
    head[fw], head[bw] = pv, pu
    cap[fw], cap[bw] = pc, prc
    rev[fw], rev[bw] = bw, fw
    return first_out, head, rev, cap, fw


@dataclass
class FlowNetwork:
    """flownet.py:41-89 FlowNetwork.

    Grid networks (:func:`build_network`) keep the int32 CUDA data volume
    ``(rows, cols, m)``, the energy parameters and the optional int32 windows
    ``lo``/``hi``; they are solved by the implicit-graph kernel.  Node numbering
    follows the reference: chain nodes site-major (node_base = cumsum(hi - lo)),
    then source, then sink.  The CSR attributes are materialised from the device
    graph on first use (module docstring).  Generic networks
    (:func:`network_from_arcs`) carry only the CSR arrays.
    """

    volume: Optional[torch.Tensor] = None
    params: Optional[EnergyParams] = None
    lo: Optional[torch.Tensor] = None
    hi: Optional[torch.Tensor] = None
    n_nodes: int = 0
    num_arcs: int = 0
    const_offset: int = 0
    # filled by a solve
    labels_dev: Optional[torch.Tensor] = field(default=None, repr=False)
    last_stats: Optional[dict] = field(default=None, repr=False)
    # explicit form (generic networks, or a materialised grid network)
    _csr: Optional[dict] = field(default=None, repr=False)
    _terminals: Optional[tuple] = field(default=None, repr=False)
    _solved_state: Optional[tuple] = field(default=None, repr=False)   # (workspace, generation) of the last grid solve

    @property
    def is_grid(self) -> bool:
        return self.volume is not None

    @property
    def site_shape(self) -> Optional[tuple[int, int]]:
        return (int(self.volume.shape[0]), int(self.volume.shape[1])) if self.is_grid else None

    @property
    def num_labels(self) -> Optional[int]:
        return int(self.volume.shape[2]) if self.is_grid else None

    @property
    def source(self) -> int:
        return self._terminals[0] if self._terminals else self.n_nodes - 2

    @property
    def sink(self) -> int:
        return self._terminals[1] if self._terminals else self.n_nodes - 1

    @property
    def has_chains(self) -> bool:
        return self.is_grid

    @property
    def materialized(self) -> bool:
        return self._csr is not None

    def windows(self):
        rows, cols = self.site_shape
        if self.lo is None:
            lo, hi = full_windows((rows, cols), self.num_labels)
            return lo.reshape(rows, cols), hi.reshape(rows, cols)
        return (self.lo.view(rows, cols).cpu().numpy(), self.hi.view(rows, cols).cpu().numpy())

    # -- the reference's CSR attributes -------------------------------------
    def materialize(self) -> dict:
        """The explicit CSR form (exported from the device graph for grid networks)."""
        if self._csr is None:
            self._csr = _export_grid_csr(self)
        return self._csr

    first_out = property(lambda self: self.materialize()["first_out"])
    head = property(lambda self: self.materialize()["head"])
    rev = property(lambda self: self.materialize()["rev"])
    cap = property(lambda self: self.materialize()["cap"])
    node_base = property(lambda self: self.materialize().get("node_base") if self.is_grid else None)
    chain_arcs = property(lambda self: self.materialize().get("chain_arcs") if self.is_grid else None)
    chain_base = property(lambda self: self.materialize().get("chain_base") if self.is_grid else None)

    @property
    def resid(self) -> np.ndarray:
        """Residual capacities.  After an implicit-graph solve this is the
        solver's final state carried to a maximum flow: the preflow it left
        (gz_export_arcs, residual mode) with the excess returned to the source
        by the CSR kernel's phase 2 -- what the reference's solver leaves."""
        return self.materialize()["resid"]

    def reset(self) -> None:
        """flownet.py:81-83: forget all flow (the device state is rebuilt by every grid solve)."""
        self.labels_dev = None
        self.last_stats = None
        self._solved_state = None
        if self._csr is not None:
            self._csr["resid"][:] = self._csr["cap"]

    def flow_sent(self) -> int:
        """flownet.py:85-89: net flow currently arriving at the sink."""
        a0, a1 = int(self.first_out[self.sink]), int(self.first_out[self.sink + 1])
        return int(-(self.cap[a0:a1] - self.resid[a0:a1]).sum())


def _export_pairs(net: FlowNetwork, residual: bool, ws=None):
    """gz_export_arcs: (pu, pv, cap, rcap) as host int64 arrays, info."""
    import ctypes as C

    from . import _lib
    rows, cols = net.site_shape
    m = net.num_labels
    L = _lib.lib()
    nbytes = L.gz_workspace_bytes(rows, cols, m)
    if ws is None:
        ws = _dev.workspace(nbytes)
    en = net.params._c()
    lo = _dev.ptr(net.lo) if net.lo is not None else None
    hi = _dev.ptr(net.hi) if net.hi is not None else None
    info = (C.c_int64 * 4)()
    vol = None if residual else _dev.ptr(net.volume)
    rc = L.gz_export_arcs(vol, rows, cols, m, C.byref(en), lo, hi, int(residual), None, None, None, None, 0, info,
                          _dev.ptr(ws), nbytes, _dev.stream_ptr())
    _lib.check(rc, "gz_export_arcs")
    npairs = int(info[0])
    buf = torch.empty((4, max(npairs, 1)), dtype=torch.int64, device=net.volume.device)
    if npairs:
        rc = L.gz_export_arcs(vol, rows, cols, m, C.byref(en), lo, hi, int(residual), _dev.ptr(buf[0]),
                              _dev.ptr(buf[1]), _dev.ptr(buf[2]), _dev.ptr(buf[3]), npairs, info, _dev.ptr(ws),
                              nbytes, _dev.stream_ptr())
        _lib.check(rc, "gz_export_arcs")
    host = buf[:, :npairs].cpu().numpy()
    return host, [int(x) for x in info]


def _export_grid_csr(net: FlowNetwork) -> dict:
    """Materialise a grid network from the device graph (flownet.py:233-296
    layout).  If the network was just solved by the implicit kernel, its final
    state is read first (the capacity export reinitialises the workspace) and
    becomes ``resid``, carried to a maximum flow (:func:`_complete_flow`)."""
    solved = None
    if net._solved_state is not None:
        ws, gen = net._solved_state
        net._solved_state = None
        if gen != _dev.workspace_generation():
            raise RuntimeError("the solve state was overwritten by a later device call; re-solve the network")
        solved = _export_pairs(net, residual=True, ws=ws)[0]
    (pu, pv, pc, prc), info = _export_pairs(net, residual=False)
    npairs, folded, n_nodes, dev_offset = info
    if folded != dev_offset or n_nodes != net.n_nodes or folded != net.const_offset:
        raise AssertionError(f"device graph export disagrees with itself: offset export {folded}, "
                             f"init {dev_offset}, model {net.const_offset}; nodes {n_nodes} vs {net.n_nodes}")
    first_out, head, rev, cap, pair_arc = pairs_to_csr(n_nodes, pu, pv, pc, prc)
    lo, hi = (a.reshape(-1).astype(np.int32) for a in net.windows())
    widths = (hi - lo).astype(np.int64)
    node_base = np.zeros(widths.size + 1, np.int64)
    np.cumsum(widths, out=node_base[1:])
    chain_base = np.zeros(widths.size + 1, np.int64)
    np.cumsum((widths + 1) * (widths > 0), out=chain_base[1:])
    # chain pairs are the ones with an UNCUTTABLE reverse (flownet.py:131), in emission order
    chain_arcs = pair_arc[prc == UNCUTTABLE].astype(np.int32)
    if chain_arcs.size != int(chain_base[-1]):
        raise AssertionError("chain arcs of the exported graph do not match the windows")
    csr = dict(first_out=first_out, head=head, rev=rev, cap=cap, resid=cap.copy(), pair_arc=pair_arc,
               node_base=node_base, chain_arcs=chain_arcs, chain_base=chain_base, lo=lo, hi=hi)
    if solved is not None:
        spu, spv, fwd, bwd = solved
        if not (np.array_equal(spu, pu) and np.array_equal(spv, pv)):
            raise AssertionError("residual export enumerates different arc pairs than the capacity export")
        csr["resid"][pair_arc] = fwd
        csr["resid"][rev[pair_arc]] = bwd
        net._csr = csr
        _complete_flow(net)
    return csr


def _complete_flow(net: FlowNetwork) -> None:
    """The implicit solver stops after phase 1, leaving a maximum
    PREflow.  Phase 2 (maxflow.py:440-457 with n + source-distance heights) on
    the CSR kernel returns the leftover excess to the source, so ``resid`` is a
    maximum flow like the reference's; the flow value must not change."""
    from .maxflow import _csr_solve
    st = _csr_solve(net, rounds_per_sweep=12, max_sweeps=None, want_side=False)[0]
    want = None if net.last_stats is None else net.last_stats.get("flow")
    if want is not None and int(st.flow) != int(want):
        raise AssertionError(f"phase-2 completion changed the flow: {int(st.flow)} != {want}")


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


def network_from_arcs(n_nodes: int, source: int, sink: int, arcs) -> FlowNetwork:
    """flownet.py:325-353: a generic network from (u, v, cap) or (u, v, cap, rcap)
    tuples; solved on the device by the CSR kernel (gz_maxflow_csr)."""
    npairs = len(arcs)
    pu = np.empty(npairs, np.int64)
    pv = np.empty(npairs, np.int64)
    pc = np.empty(npairs, np.int64)
    prc = np.zeros(npairs, np.int64)
    for i, arc in enumerate(arcs):
        u, v, c = arc[0], arc[1], arc[2]
        if not (0 <= u < n_nodes and 0 <= v < n_nodes):
            raise ValueError(f"arc ({u}, {v}) outside node range")
        if c < 0 or (len(arc) > 3 and arc[3] < 0):
            raise ValueError("negative capacity")
        pu[i], pv[i], pc[i] = u, v, c
        if len(arc) > 3:
            prc[i] = arc[3]
    first_out, head, rev, cap, pair_arc = pairs_to_csr(n_nodes, pu, pv, pc, prc)
    csr = dict(first_out=first_out, head=head, rev=rev, cap=cap, resid=cap.copy(), pair_arc=pair_arc)
    return FlowNetwork(n_nodes=n_nodes, num_arcs=int(head.size), _csr=csr, _terminals=(source, sink))


def node_blocks(net: FlowNetwork, block: int) -> np.ndarray:
    """flownet.py:356-382: level-2 scheduling block of every node (terminals 0).
    The device's capped schedule is the GPU's own; this is the
    reference's block key, for callers that order work by it."""
    if not net.has_chains:
        raise ValueError("network has no chain metadata")
    rows, cols = net.site_shape
    m = net.num_labels
    gb, mb = -(-cols // block), -(-m // block)
    lo, hi = (a.reshape(-1).astype(np.int64) for a in net.windows())
    widths = hi - lo
    site = np.repeat(np.arange(rows * cols), widths)
    start = np.repeat(np.cumsum(widths) - widths, widths)
    t = lo[site] + 1 + (np.arange(site.size) - start)
    y, g = site // cols, site % cols
    out = np.zeros(net.n_nodes, np.int32)
    out[: site.size] = (y // block) * gb * mb + (g // block) * mb + t // block
    return out


def dump_network(net: FlowNetwork, file) -> None:
    """flownet.py:385-397: header line, then ``tail head cap`` per arc in CSR order."""
    file.write(f"nodes {net.n_nodes} source {net.source} sink {net.sink} offset {net.const_offset}\n")
    fo, head, cap = net.first_out, net.head, net.cap
    for u in range(net.n_nodes):
        for a in range(int(fo[u]), int(fo[u + 1])):
            file.write(f"{u} {int(head[a])} {int(cap[a])}\n")
