"""The reference's own hot-path unit tests, adapted to run against this
package on the GPU (the reference is absent on the GPU box, so each case is
restated here with its source line; brute-force oracles are small Python
loops or the C oracle).  Sources: pkg/tests/test_maxflow.py,
test_flownet.py, test_energy.py, test_hierarchy.py."""

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _random_net(rng, n_max=24, cap_max=20):
    """test_maxflow.py:18-29."""
    n = int(rng.integers(4, n_max))
    arcs = [(u, u + 1, int(rng.integers(0, cap_max))) for u in range(n - 1)]
    for _ in range(int(rng.integers(n, 4 * n))):
        u, v = rng.integers(0, n, 2)
        if u != v:
            arcs.append((int(u), int(v), int(rng.integers(0, cap_max))))
    return n, arcs


def _cut_capacity(net, side):
    """test_maxflow.py:32-40."""
    total = 0
    for u in range(net.n_nodes):
        if side[u]:
            for a in range(int(net.first_out[u]), int(net.first_out[u + 1])):
                if not side[net.head[a]]:
                    total += int(net.cap[a])
    return total


def _plain_energy(lab, vol, p):
    """oracle.py:15-33 plain_energy (total_energy by loops)."""
    from paper_1803_01516_b200.energy import pairwise_term
    rows, cols, _ = vol.shape
    e = sum(int(vol[y, g, lab[y, g]]) for y in range(rows) for g in range(cols))
    for y in range(rows):
        for g in range(cols):
            if g + 1 < cols:
                e += pairwise_term(int(lab[y, g]), int(lab[y, g + 1]), p)
            if y + 1 < rows:
                e += pairwise_term(int(lab[y, g]), int(lab[y + 1, g]), p)
    return e


def _exhaustive(vol, p, lo=None, hi=None):
    rows, cols, m = vol.shape
    ranges = [range(m)] * (rows * cols) if lo is None else [range(lo[s], hi[s] + 1) for s in range(rows * cols)]
    return min(_plain_energy(np.array(c).reshape(rows, cols), vol, p) for c in itertools.product(*ranges))


# ---- test_maxflow.py -------------------------------------------------------

def test_solvers_agree_on_random_networks(gz, oracle):
    """test_maxflow.py:43-50: Dinic = push-relabel = plain max flow (120 nets)."""
    rng = np.random.default_rng(31)
    for _ in range(120):
        n, arcs = _random_net(rng)
        f_ref = gz.maxflow_reference(gz.network_from_arcs(n, 0, n - 1, arcs)).flow
        f_pr = gz.maxflow_push_relabel(gz.network_from_arcs(n, 0, n - 1, arcs)).flow
        f_oracle = oracle.maxflow_dinic(oracle.network_from_arcs(n, 0, n - 1, arcs))[0]
        assert f_ref == f_pr == f_oracle


def test_flow_matches_scipy(gz):
    """test_maxflow.py:53-65."""
    sparse = pytest.importorskip("scipy.sparse")
    from scipy.sparse.csgraph import maximum_flow
    rng = np.random.default_rng(32)
    for _ in range(40):
        n, arcs = _random_net(rng)
        dense = np.zeros((n, n), dtype=np.int32)
        for u, v, c in arcs:
            dense[u, v] += c
        want = maximum_flow(sparse.csr_matrix(dense), 0, n - 1).flow_value
        assert gz.maxflow_reference(gz.network_from_arcs(n, 0, n - 1, arcs)).flow == want


def test_flow_conservation_and_cut_capacity(gz):
    """test_maxflow.py:68-78."""
    from paper_1803_01516_b200.maxflow import conservation_violations
    rng = np.random.default_rng(33)
    for _ in range(60):
        n, arcs = _random_net(rng)
        net = gz.network_from_arcs(n, 0, n - 1, arcs)
        r = gz.maxflow_push_relabel(net)
        assert conservation_violations(net) == 0
        assert r.flow == _cut_capacity(net, r.source_side)
        assert r.source_side[net.source] and not r.source_side[net.sink]


def test_gaze_networks_yield_identical_labelings(gz):
    """test_maxflow.py:81-95: both exact solvers, the same canonical cut."""
    rng = np.random.default_rng(34)
    for _ in range(40):
        rows, cols, m = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(2, 6))
        vol = rng.integers(0, 90, (rows, cols, m)).astype(np.int64)
        p = gz.EnergyParams(penalty=int(rng.integers(0, 6)), inhibit=int(rng.integers(0, 40)))
        a = gz.solve_exact(vol, p, solver="dinic")
        b = gz.solve_exact(vol, p, solver="push-relabel")
        assert a.flow == b.flow and a.energy == b.energy
        assert np.array_equal(a.labeling, b.labeling)


def test_exact_energy_matches_exhaustive_minimum(gz):
    """test_maxflow.py:98-112."""
    rng = np.random.default_rng(35)
    for _ in range(25):
        m = int(rng.integers(2, 5))
        vol = rng.integers(0, 70, (2, 2, m)).astype(np.int64)
        p = gz.EnergyParams(penalty=int(rng.integers(1, 5)), inhibit=int(rng.integers(0, 25)))
        best = _exhaustive(vol, p)
        r = gz.solve_exact(vol, p)
        assert r.energy == best == _plain_energy(r.labeling, vol, p)


def test_presaturation_changes_nothing_observable(gz):
    """test_maxflow.py:115-128 (grid networks: the implicit kernel)."""
    rng = np.random.default_rng(36)
    for _ in range(15):
        vol = rng.integers(0, 90, (2, 3, 4)).astype(np.int64)
        p = gz.EnergyParams(3, 12)
        r1 = gz.maxflow_push_relabel(gz.build_network(vol, p), presaturate=True)
        r2 = gz.maxflow_push_relabel(gz.build_network(vol, p), presaturate=False)
        assert (r1.flow, r1.energy) == (r2.flow, r2.energy)
        assert np.array_equal(r1.labeling, r2.labeling)
        assert r1.stats["presaturated"] > 0 and r2.stats["presaturated"] == 0


def test_presaturation_on_explicit_networks(gz):
    """The same on materialised networks (chain_presaturate + the CSR kernel)."""
    rng = np.random.default_rng(36)
    for _ in range(6):
        vol = rng.integers(1, 90, (2, 3, 4)).astype(np.int64)
        p = gz.EnergyParams(3, 12)
        n1, n2 = gz.build_network(vol, p), gz.build_network(vol, p)
        n1.materialize(), n2.materialize()
        r1 = gz.maxflow_push_relabel(n1, presaturate=True)
        r2 = gz.maxflow_push_relabel(n2, presaturate=False)
        assert (r1.flow, r1.energy) == (r2.flow, r2.energy)
        assert np.array_equal(r1.labeling, r2.labeling)
        assert r1.stats["presaturated"] > 0 and r2.stats["presaturated"] == 0


def test_chain_presaturate_is_feasible(gz):
    """test_maxflow.py:131-139."""
    from paper_1803_01516_b200.maxflow import chain_presaturate, conservation_violations
    rng = np.random.default_rng(37)
    vol = rng.integers(1, 90, (2, 3, 5)).astype(np.int64)
    net = gz.build_network(vol, gz.EnergyParams(3, 12))
    sent = chain_presaturate(net)
    assert sent >= vol.min(axis=2).sum()
    assert (net.resid >= 0).all()
    assert conservation_violations(net) == 0


def test_solver_stats_fields(gz):
    """test_maxflow.py:142-158."""
    vol = np.random.default_rng(38).integers(0, 50, (2, 2, 3)).astype(np.int64)
    p = gz.EnergyParams(2, 7)
    r = gz.solve_exact(vol, p)
    for key in ("solver", "wall_s", "converged", "sweeps", "pushes", "relabels", "presaturated",
                "stranded_excess_nodes", "build_s", "nodes", "arcs", "const_offset"):
        assert key in r.stats
    assert r.stats["solver"] == "push-relabel"
    assert r.stats["converged"] is True
    assert r.stats["stranded_excess_nodes"] == 0
    d = gz.solve_exact(vol, p, solver="dinic")
    assert d.stats["solver"] == "dinic" and d.stats["stranded_excess_nodes"] == 0
    with pytest.raises(ValueError):
        gz.solve_exact(vol, p, solver="bogus")
    with pytest.raises(ValueError):
        gz.maxflow_push_relabel(gz.build_network(vol, p), rounds_per_sweep=0)


def test_stranded_excess_is_zero_and_deterministic_on_c1(gz):
    """stranded_excess_nodes was the phase-1 leftover (~317k on C1,
    nondeterministic).  A converged solve strands nothing (maxflow.py:460-471)."""
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    sc = gz.make_scene(0)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    for _ in range(2):
        assert gz.solve_exact(vol, gz.EnergyParams(14, 1023)).stats["stranded_excess_nodes"] == 0


def test_sweep_cap_reports_unconverged(gz):
    """test_maxflow.py:161-173."""
    rng = np.random.default_rng(39)
    vol = rng.integers(0, 200, (4, 5, 6)).astype(np.int64)
    p = gz.EnergyParams(5, 50)
    r = gz.maxflow_push_relabel(gz.build_network(vol, p), rounds_per_sweep=1, max_sweeps=1)
    if not r.stats["converged"]:
        assert r.energy is None and r.stats["sweeps"] == 1
    exact = gz.maxflow_push_relabel(gz.build_network(vol, p))
    assert exact.stats["converged"]
    assert exact.flow >= r.flow or not r.stats["converged"]


# ---- test_flownet.py -------------------------------------------------------

def test_count_formulas_match_built_networks(gz):
    """test_flownet.py:72-79, on the exported device graph."""
    rng = np.random.default_rng(21)
    for rows, cols in [(1, 1), (1, 2), (2, 2), (3, 4), (2, 5)]:
        for m in [2, 3, 5, 7]:
            vol = rng.integers(0, 100, (rows, cols, m)).astype(np.int64)
            net = gz.build_network(vol, gz.EnergyParams(2, 9))
            assert net.n_nodes == gz.expected_node_count((rows, cols), m)
            assert net.num_arcs == int(net.head.size) == gz.expected_arc_count((rows, cols), m)


def test_window_validation(gz):
    """test_flownet.py:99-108."""
    vol = np.zeros((1, 2, 3), dtype=np.int64)
    p = gz.EnergyParams()
    lo, hi = gz.full_windows((1, 2), 3)
    for a, b in ((hi, lo), (lo - 1, hi), (lo, hi + 1)):
        with pytest.raises(ValueError):
            gz.build_network(vol, p, lo=a, hi=b)


def test_fully_forced_windows_fold_into_offset(gz):
    """test_flownet.py:111-124."""
    rng = np.random.default_rng(23)
    for _ in range(20):
        vol = rng.integers(0, 60, (2, 3, 4)).astype(np.int64)
        p = gz.EnergyParams(penalty=int(rng.integers(0, 5)), inhibit=int(rng.integers(0, 30)))
        lab = rng.integers(0, 4, (2, 3)).astype(np.int32)
        net = gz.build_network(vol, p, lo=lab, hi=lab)
        assert net.n_nodes == 2
        r = gz.maxflow_reference(net)
        assert r.flow == 0 and r.energy == _plain_energy(lab, vol, p)
        assert np.array_equal(r.labeling, lab)


def test_restricted_windows_match_windowed_brute_force(gz):
    """test_flownet.py:127-150."""
    rng = np.random.default_rng(24)
    for _ in range(25):
        vol = rng.integers(0, 60, (2, 2, 4)).astype(np.int64)
        p = gz.EnergyParams(penalty=int(rng.integers(1, 5)), inhibit=int(rng.integers(0, 30)))
        lo = rng.integers(0, 4, 4).astype(np.int32)
        hi = np.minimum(lo + rng.integers(0, 4, 4), 3).astype(np.int32)
        lo = np.minimum(lo, hi)
        r = gz.maxflow_reference(gz.build_network(vol, p, lo=lo, hi=hi))
        assert r.energy == _exhaustive(vol, p, lo, hi)
        flat = r.labeling.reshape(-1)
        assert (flat >= lo).all() and (flat <= hi).all()
        # the implicit kernel on the same windows
        r2 = gz.maxflow_push_relabel(gz.build_network(vol, p, lo=lo, hi=hi))
        assert r2.energy == r.energy and np.array_equal(r2.labeling, r.labeling)


def test_single_label_volume(gz):
    """test_flownet.py:153-158."""
    vol = np.arange(6, dtype=np.int64).reshape(2, 3, 1)
    net = gz.build_network(vol, gz.EnergyParams(3, 7))
    assert net.n_nodes == 2 and net.num_arcs == 0 and net.const_offset == vol.sum()


def test_network_from_arcs_classic(gz):
    """test_flownet.py:161-175: textbook flows 5 and 3."""
    net = gz.network_from_arcs(4, 0, 3, [(0, 1, 3), (0, 2, 2), (1, 2, 1), (1, 3, 2), (2, 3, 3)])
    assert gz.maxflow_reference(net).flow == 5
    assert gz.maxflow_reference(gz.network_from_arcs(3, 0, 2, [(0, 1, 4, 1), (1, 2, 3, 2)])).flow == 3


def test_node_blocks_tiling(gz, oracle):
    """test_flownet.py:178-190 (node_blocks against the oracle)."""
    from paper_1803_01516_b200.flownet import node_blocks
    rng = np.random.default_rng(25)
    vol = rng.integers(0, 50, (4, 5, 6)).astype(np.int64)
    for b in (1, 2, 3):
        got = node_blocks(gz.build_network(vol, gz.EnergyParams()), b)
        want = oracle.node_blocks(oracle.build_network(vol, 14, 1023), b)
        assert np.array_equal(got, want)


# ---- test_energy.py --------------------------------------------------------

def test_pairwise_table(gz):
    """test_energy.py:20-28."""
    p = gz.EnergyParams(14, 1023)
    pt = gz.pairwise_term
    assert (pt(4, 4, p), pt(4, 5, p), pt(5, 4, p)) == (0, 14, 14)
    assert pt(4, 6, p) == pt(6, 4, p) == 2 * 14 + 1023
    assert pt(0, 3, p) == 3 * 14 + 2 * 1023 and pt(0, 5, p) == 5 * 14 + 4 * 1023


def test_sad_volume_matches_direct_lookup(gz):
    """test_energy.py:66-87 (200 random probes)."""
    width, height = 40, 6
    c = gz.cuboid_from_disparity_range(width, height, 5, 13)
    rng = np.random.default_rng(7)
    left = rng.integers(0, 256, (height, width, 3)).astype(np.uint8)
    right = rng.integers(0, 256, (height, width, 3)).astype(np.uint8)
    vol = gz.sad_volume(left, right, c)
    assert vol.shape == (c.y_extent, c.g_extent, c.num_labels) and vol.dtype == np.int64
    assert vol.min() >= 0 and vol.max() <= 765
    li, ri = np.int64(left), np.int64(right)
    for _ in range(200):
        yi, gi, t = int(rng.integers(0, c.y_extent)), int(rng.integers(0, c.g_extent)), int(rng.integers(0, c.num_labels))
        g, d = c.g_min + gi, c.d_min + t
        xr, xl = min(max(g + d, 0), width - 1), min(max(width - 1 + g - d, 0), width - 1)
        assert vol[yi, gi, t] == int(np.abs(li[yi, xl] - ri[yi, xr]).sum())


def test_sad_volume_greyscale_and_shape_mismatch(gz):
    """test_energy.py:90-98."""
    c = gz.cuboid_from_disparity_range(16, 3, 1, 5)
    rng = np.random.default_rng(8)
    left = rng.integers(0, 256, (3, 16)).astype(np.uint8)
    right = rng.integers(0, 256, (3, 16)).astype(np.uint8)
    assert gz.sad_volume(left, right, c).max() <= 255
    with pytest.raises(ValueError):
        gz.sad_volume(left, right[:2], c)


def test_total_energy_matches_plain_energy(gz):
    """test_energy.py:101-144 family: total_energy (device) = plain loops, incl. hard."""
    rng = np.random.default_rng(9)
    for _ in range(20):
        rows, cols, m = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 6))
        vol = rng.integers(0, 100, (rows, cols, m)).astype(np.int64)
        p = gz.EnergyParams(int(rng.integers(0, 9)), int(rng.integers(0, 50)), bool(rng.integers(0, 2)))
        lab = rng.integers(0, m, (rows, cols)).astype(np.int32)
        want = _plain_energy(lab, vol, p)
        got = gz.total_energy(lab, vol, p)
        assert got == (gz.UNCUTTABLE if want >= gz.UNCUTTABLE else want)


# ---- test_hierarchy.py -----------------------------------------------------

def test_coarsen_hand_case(gz):
    """test_hierarchy.py:9-18."""
    vol = np.arange(2 * 4 * 4, dtype=np.int64).reshape(2, 4, 4)
    coarse, cp = gz.coarsen(vol, 2, gz.EnergyParams(5, 99))
    assert coarse.shape == (1, 2, 2) and coarse[0, 0, 0] == vol[0:2, 0:2, 0:2].sum()
    assert (cp.penalty, cp.inhibit) == (10, 99)


def test_coarsen_zero_pads_ragged_shapes(gz):
    """test_hierarchy.py:21-28."""
    vol = np.ones((3, 5, 3), dtype=np.int64)
    coarse, _ = gz.coarsen(vol, 2, gz.EnergyParams())
    assert coarse.shape == (2, 3, 2) and coarse.sum() == vol.sum() and coarse[1, 2, 1] == 1
    with pytest.raises(ValueError):
        gz.coarsen(vol, 0, gz.EnergyParams())


def test_thin_skin_frozen_values(gz):
    """test_hierarchy.py:31-40."""
    lo, hi = gz.thin_skin(np.array([[0, 2], [1, 3]]), (4, 4, 12), block=3, radius=1)
    assert lo.shape == hi.shape == (4, 4)
    assert (lo[0, 0], hi[0, 0], lo[0, 3], hi[0, 3]) == (0, 5, 3, 11)
    assert (lo[3, 0], hi[3, 0], lo[3, 3], hi[3, 3]) == (0, 8, 6, 11)
    assert (lo <= hi).all()


def test_level1_block1_is_bit_identical_to_exact(gz):
    """test_hierarchy.py:52-59."""
    vol = np.random.default_rng(42).integers(0, 120, (5, 6, 7)).astype(np.int64)
    p = gz.EnergyParams(6, 30)
    e, l1 = gz.solve_exact(vol, p), gz.solve_level1(vol, p, block=1)
    assert l1.energy == e.energy and np.array_equal(l1.labeling, e.labeling)


def test_hierarchy_energies_are_monotone(gz):
    """test_hierarchy.py:62-71."""
    rng = np.random.default_rng(43)
    for _ in range(5):
        vol = rng.integers(0, 300, (8, 9, 8)).astype(np.int64)
        p = gz.EnergyParams(7, 60)
        e0 = gz.solve_exact(vol, p).energy
        e1 = gz.solve_level1(vol, p, block=2).energy
        e2 = gz.solve_level2(vol, p, block=2, max_sweeps=1).energy
        assert e0 <= e1 <= e2


def test_level2_uncapped_equals_level1(gz):
    """test_hierarchy.py:74-82."""
    vol = np.random.default_rng(44).integers(0, 200, (6, 7, 9)).astype(np.int64)
    p = gz.EnergyParams(5, 40)
    l1 = gz.solve_level1(vol, p, block=3)
    l2 = gz.solve_level2(vol, p, block=3, max_sweeps=None)
    assert l2.energy == l1.energy and np.array_equal(l2.labeling, l1.labeling) and l2.stats["converged"]


def test_level_stats_shape(gz):
    """test_hierarchy.py:85-96."""
    vol = np.random.default_rng(45).integers(0, 100, (4, 4, 6)).astype(np.int64)
    p = gz.EnergyParams(4, 25)
    l1 = gz.solve_level1(vol, p, block=2)
    assert (l1.stats["level"], l1.stats["block"]) == (1, 2)
    assert l1.stats["mean_window"] <= 6.0 and l1.stats["coarse_energy"] >= 0
    l2 = gz.solve_level2(vol, p, block=2)
    assert l2.stats["level"] == 2 and "wall_s" in l2.stats and "coarse_wall_s" in l2.stats
    d = gz.solve_level1(vol, p, block=2, solver="dinic")
    assert d.stats["solver"] == "dinic" and d.energy == l1.energy and np.array_equal(d.labeling, l1.labeling)


def test_labels_stay_inside_skin(gz):
    """test_hierarchy.py:99-107."""
    vol = np.random.default_rng(46).integers(0, 150, (6, 6, 10)).astype(np.int64)
    p = gz.EnergyParams(3, 20)
    cvol, cp = gz.coarsen(vol, 2, p)
    coarse = gz.solve_exact(cvol, cp)
    lo, hi = gz.thin_skin(coarse.labeling, vol.shape, 2, 1)
    l1 = gz.solve_level1(vol, p, block=2)
    assert (l1.labeling >= lo).all() and (l1.labeling <= hi).all()
