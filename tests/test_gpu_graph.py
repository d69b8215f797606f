"""The DEVICE graph against the reference's explicit construction
(flownet.py:102-296).  gz_export_arcs runs the solver's own initialisation
and enumerates the implicit graph's arc pairs in _emit order with capacities
read from the initialised state planes; FlowNetwork lays them out as CSR
(pairs_to_csr = flownet.py:184-222).  Checked against the reference's golden
1x2x3 dump (pkg/tests/test_flownet.py:28-61), its chain capacities
(test_flownet.py:64-69) and its CSR arrays for the 90 random golden cases
(plain, windowed, hard inhibit; tests/golden/csr.json)."""

import hashlib
import io
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLDEN / "golden.json").read_text())
CSR = json.loads((GOLDEN / "csr.json").read_text())["cases"]


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=dtype)).tobytes()).hexdigest()


def test_golden_dump_from_the_device_graph(gz):
    from paper_1803_01516_b200.flownet import dump_network
    net = gz.build_network(np.array([[[5, 7, 9], [6, 8, 10]]], np.int64), gz.EnergyParams(3, 11))
    buf = io.StringIO()
    dump_network(net, buf)
    assert buf.getvalue() == G["golden_1x2x3_dump"]


def test_golden_chain_arc_capacities(gz):
    net = gz.build_network(np.array([[[5, 7, 9], [6, 8, 10]]], np.int64), gz.EnergyParams(3, 11))
    assert net.chain_base.tolist() == [0, 3, 6]
    caps = net.cap[net.chain_arcs]
    assert caps[0:3].tolist() == [5, 7, 9] and caps[3:6].tolist() == [6, 8, 10]


def test_random_cases_csr_equal_the_reference(gz):
    arr = np.load(GOLDEN / "random_cases.npz")
    for i, meta in enumerate(G["random_cases"]):
        lo = arr[f"lo{i}"] if meta["windowed"] else None
        hi = arr[f"hi{i}"] if meta["windowed"] else None
        net = gz.build_network(arr[f"vol{i}"], gz.EnergyParams(meta["penalty"], meta["inhibit"], meta["hard"]), lo, hi)
        want = CSR[i]
        assert (net.n_nodes, net.const_offset) == (want["nodes"], want["const_offset"]), i
        assert int(net.head.size) == want["arcs"] == net.num_arcs, i
        for k, dt in (("first_out", np.int64), ("head", np.int32), ("rev", np.int32), ("cap", np.int64),
                      ("node_base", np.int64), ("chain_arcs", np.int32), ("chain_base", np.int64)):
            assert sha(getattr(net, k), dt) == want[k], (i, k, meta)


@pytest.mark.parametrize("m", [3, 17, 40, 129])
def test_structural_invariants_device_graph(gz, m):
    """pkg/tests/test_flownet.py:82-96 on exported graphs of every chain layout
    (16-lane, one/two/five 32-lane segments)."""
    rng = np.random.default_rng(22 + m)
    vol = rng.integers(0, 80, (3, 4, m)).astype(np.int64)
    net = gz.build_network(vol, gz.EnergyParams(4, 17))
    n, fo = net.n_nodes, net.first_out
    assert n == gz.expected_node_count((3, 4), m) and net.head.size == gz.expected_arc_count((3, 4), m)
    assert fo[0] == 0 and fo[n] == net.head.size and (np.diff(fo) >= 0).all()
    owner = np.repeat(np.arange(n), np.diff(fo))
    assert np.array_equal(net.rev[net.rev], np.arange(net.head.size))
    assert np.array_equal(net.head[net.rev], owner)
    assert (net.cap >= 0).all() and np.array_equal(net.resid, net.cap)
    assert (net.head != owner).all() and net.head.min() >= 0 and net.head.max() < n
    # the explicit graph solved by the CSR kernel equals the implicit solve
    implicit = gz.solve_exact(vol, gz.EnergyParams(4, 17))
    explicit = gz.maxflow_push_relabel(net)
    assert explicit.flow == implicit.flow and np.array_equal(explicit.labeling, implicit.labeling)


def test_c1_device_graph_counts_and_capacities(gz, oracle):
    """A full C1 graph (1.6 M nodes, 21.8 M arcs): the device export equals the
    oracle's explicit construction arc for arc."""
    sc = gz.make_scene(0)
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    net = gz.build_network(vol, gz.EnergyParams(14, 1023))
    ref = oracle.build_network(vol, 14, 1023)
    for k in ("first_out", "head", "rev", "cap", "node_base", "chain_arcs", "chain_base"):
        assert np.array_equal(getattr(net, k), getattr(ref, k)), k
    assert net.n_nodes == 1607042 and net.head.size == 21798984


def test_solved_grid_state_is_a_maximum_flow(gz, oracle):
    """After an implicit solve, ``resid`` is the solver's final preflow
    (gz_export_arcs residual mode) carried to a maximum flow by the CSR
    kernel's phase 2: conservation holds, the flow is unchanged and its
    source side is the labeling's."""
    from paper_1803_01516_b200.maxflow import conservation_violations
    rng = np.random.default_rng(40)
    for m in (5, 24, 70):
        vol = rng.integers(0, 120, (7, 9, m)).astype(np.int64)
        p = gz.EnergyParams(5, 30)
        net = gz.build_network(vol, p)
        r = gz.maxflow_push_relabel(net)
        assert conservation_violations(net) == 0
        assert net.flow_sent() == r.flow
        assert (net.resid >= 0).all()
        side = gz.source_side(net)
        assert np.array_equal(gz.extract_labeling(net, side), r.labeling)
