"""Bit-exact parity of the sm_100a path with the CPU oracle (oracle/gz_oracle.c,
itself pinned to the reference in test_oracle.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand_cases(seed, n, max_side=7, max_m=8, windows=False):
    rng = np.random.default_rng(seed)
    for i in range(n):
        rows, cols, m = int(rng.integers(1, max_side)), int(rng.integers(1, max_side)), int(rng.integers(2, max_m))
        vol = rng.integers(0, 200, (rows, cols, m)).astype(np.int64)
        pen, inh, hard = int(rng.integers(0, 9)), int(rng.integers(0, 80)), bool(rng.integers(5) == 0)
        lo = hi = None
        if windows:
            lo = rng.integers(0, m, rows * cols).astype(np.int32)
            hi = np.minimum(lo + rng.integers(0, m, rows * cols), m - 1).astype(np.int32)
        yield vol, pen, inh, hard, lo, hi


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_exact_random_volumes(gz, oracle, seed):
    for vol, pen, inh, hard, _, _ in _rand_cases(seed, 40):
        p = gz.EnergyParams(pen, inh, hard)
        got = gz.solve_exact(vol, p)
        want = oracle.solve_exact(vol, pen, inh, hard)
        assert got.flow == want["flow"]
        assert got.energy == want["energy"]
        assert np.array_equal(got.labeling, want["labeling"])
        assert np.array_equal(got.source_side, want["source_side"])
        assert got.stats["nodes"] == want["stats"]["nodes"]
        assert got.stats["arcs"] == want["stats"]["arcs"]


@pytest.mark.parametrize("seed", [4, 5])
def test_windowed_random_volumes(gz, oracle, seed):
    for vol, pen, inh, hard, lo, hi in _rand_cases(seed, 40, windows=True):
        p = gz.EnergyParams(pen, inh, hard)
        net = gz.build_network(vol, p, lo, hi)
        got = gz.maxflow_push_relabel(net)
        onet = oracle.build_network(vol, pen, p.inhibit_capacity, lo, hi)
        flow, energy, lab, side, st = oracle.maxflow_push_relabel(onet)
        assert net.const_offset == onet.const_offset
        assert net.n_nodes == onet.n_nodes and net.num_arcs == onet.num_arcs
        assert got.flow == flow and got.energy == energy
        assert np.array_equal(got.labeling, lab)
        assert np.array_equal(got.source_side, side)


def test_c1_seed0(gz, oracle):
    sc = gz.make_scene(0)
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    ovol = oracle.sad_volume(sc.left, sc.right, cub.g_min, cub.g_extent, cub.y_min, cub.y_extent, cub.d_min, 16)
    assert np.array_equal(vol, ovol)
    r = gz.solve_exact(vol, gz.EnergyParams(14, 1023))
    assert r.flow == 778554 and r.energy == 778554
    want = oracle.solve_exact(ovol, 14, 1023)
    assert np.array_equal(r.labeling, want["labeling"])
    print("C1 stats", r.stats)


def test_level1_matches_oracle(gz, oracle):
    rng = np.random.default_rng(46)
    for i in range(10):
        vol = rng.integers(0, 300, (int(rng.integers(4, 12)), int(rng.integers(4, 12)), int(rng.integers(4, 12)))).astype(np.int64)
        pen, inh, b = int(rng.integers(1, 9)), int(rng.integers(0, 90)), int(rng.integers(1, 4))
        p = gz.EnergyParams(pen, inh)
        got = gz.solve_level1(vol, p, b)
        want = oracle.solve_level1(vol, pen, inh, b)
        assert got.energy == want["energy"] and got.flow == want["flow"]
        assert np.array_equal(got.labeling, want["labeling"])
        assert got.stats["coarse_energy"] == want["coarse_energy"]


def test_level2_properties(gz, oracle):
    rng = np.random.default_rng(43)
    for _ in range(5):
        vol = rng.integers(0, 300, (8, 9, 8)).astype(np.int64)
        p = gz.EnergyParams(7, 60)
        e0 = gz.solve_exact(vol, p).energy
        l1 = gz.solve_level1(vol, p, 2)
        l2 = gz.solve_level2(vol, p, 2, max_sweeps=1)
        assert e0 <= l1.energy <= l2.energy
        l2u = gz.solve_level2(vol, p, 2, max_sweeps=None)
        assert l2u.energy == l1.energy and np.array_equal(l2u.labeling, l1.labeling)


def test_c1_level1(gz, oracle):
    sc = gz.make_scene(0)
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    for b in (2, 4):
        r = gz.solve_level1(vol, gz.EnergyParams(14, 1023), b)
        want = oracle.solve_level1(vol, 14, 1023, b)
        assert r.energy == want["energy"] and np.array_equal(r.labeling, want["labeling"])
        print("C1 L1 b", b, r.energy, r.stats["device_ms"], r.stats["wall_s"])


@pytest.mark.parametrize("m", [33, 70, 129, 200, 256])
def test_long_chains_match_oracle(gz, oracle, m):
    """Chains of 2-8 warp segments (m > 32): segment-crossing waves and pushes,
    multi-word BFS (global-memory masks at m > 128), against the oracle."""
    rng = np.random.default_rng(1000 + m)
    for _ in range(3):
        rows, cols = int(rng.integers(2, 6)), int(rng.integers(2, 6))
        vol = rng.integers(0, 120, (rows, cols, m)).astype(np.int64)
        pen, inh = int(rng.integers(1, 9)), int(rng.integers(0, 60))
        got = gz.solve_exact(vol, gz.EnergyParams(pen, inh))
        want = oracle.solve_exact(vol, pen, inh)
        assert got.flow == want["flow"] and got.energy == want["energy"]
        assert np.array_equal(got.labeling, want["labeling"])


@pytest.mark.parametrize("m", [6, 24, 40])
def test_capped_solves_are_deterministic(gz, m):
    """Capped sweeps (level 2) run the GPU's own deterministic schedule: push,
    relabel into a second height buffer, commit.  Identical
    flow and labeling run to run, at every sweep cap."""
    rng = np.random.default_rng(77 + m)
    for _ in range(3):
        rows, cols = int(rng.integers(8, 30)), int(rng.integers(8, 30))
        vol = rng.integers(0, 200, (rows, cols, m)).astype(np.int64)
        p = gz.EnergyParams(int(rng.integers(1, 9)), int(rng.integers(0, 60)))
        lo = rng.integers(0, m, rows * cols).astype(np.int32)
        hi = np.minimum(lo + rng.integers(0, 6, rows * cols), m - 1).astype(np.int32)
        for cap in (1, 2, 4):
            runs = []
            for _ in range(2):
                net = gz.build_network(vol, p, lo, hi)
                r = gz.maxflow_push_relabel(net, max_sweeps=cap)
                runs.append((r.flow, r.labeling.copy(), r.stats["sweeps"], r.stats["pulses"]))
            assert runs[0][0] == runs[1][0] and np.array_equal(runs[0][1], runs[1][1]), (m, cap)
            assert runs[0][2:] == runs[1][2:]


@pytest.mark.parametrize("m", [20, 30, 45, 60])
def test_narrow_windows_match_oracle(gz, oracle, m):
    """Windows at most 15 positions wide on 17 <= m <= 64 run the window-relative
    16-lane instance (the level-1/2 fine solves); bit-exact vs the oracle."""
    rng = np.random.default_rng(500 + m)
    for k in range(4):
        rows, cols = int(rng.integers(3, 12)), int(rng.integers(3, 12))
        vol = rng.integers(0, 150, (rows, cols, m)).astype(np.int64)
        pen, inh, hard = int(rng.integers(1, 9)), int(rng.integers(0, 60)), k == 3
        p = gz.EnergyParams(pen, inh, hard)
        lo = rng.integers(0, m, rows * cols).astype(np.int32)
        hi = np.minimum(lo + rng.integers(0, 16, rows * cols), m - 1).astype(np.int32)
        net = gz.build_network(vol, p, lo, hi)
        got = gz.maxflow_push_relabel(net)
        onet = oracle.build_network(vol, pen, p.inhibit_capacity, lo, hi)
        flow, energy, lab, side, _ = oracle.maxflow_push_relabel(onet)
        assert net.const_offset == onet.const_offset
        assert got.flow == flow and got.energy == energy, (m, k)
        assert np.array_equal(got.labeling, lab) and np.array_equal(got.source_side, side)


@pytest.mark.parametrize("m,hard", [(300, False), (300, True), (400, False)])
def test_v1_solver_beyond_256_labels(gz, oracle, m, hard):
    """m > 256 runs the v1 planar column-relaxation solver (choose_solver in
    gz_solver.cu); it must agree with the reference restatement bit for bit."""
    rng = np.random.default_rng(m + hard)
    vol = rng.integers(0, 60, size=(6, 7, m)).astype(np.int64)
    p = gz.EnergyParams(3, 11, hard)
    got = gz.solve_exact(vol, p)
    want = oracle.solve_exact(vol, 3, 11, hard)
    assert got.flow == want["flow"] and got.energy == want["energy"]
    assert np.array_equal(got.labeling, want["labeling"])
    assert got.stats["stranded_excess_nodes"] == 0
