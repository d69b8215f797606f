"""Capped (level-2) solves against the CPU restatement of the device's own
deterministic schedule (oracle/gz_capped.c; the reference's
sequential FIFO schedule, maxflow.py:198-249, cannot be replayed on a GPU, so
the GPU schedule is restated and pinned bit for bit).  The restatement takes
the device's BFS blocking depth (stats['bfs_h']); pulses per sweep and the
BFS early-stop depth follow gz_solver.cu (rounds_per_sweep, max(24, m))."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _restated(oracle, vol, p, lo, hi, max_sweeps, bfs_h, rounds=12):
    m = vol.shape[2]
    return oracle.capped_schedule(vol, p.penalty, p.inhibit, lo, hi, K=rounds, max_sweeps=max_sweeps,
                                  bfs_min=max(24, m), H=bfs_h)


@pytest.mark.parametrize("m,width,max_sweeps", [(12, 3, 1), (12, 5, 2), (16, 15, 3), (24, 5, 1), (24, 8, 2),
                                                (40, 11, 4), (60, 15, 3)])
def test_capped_windowed_solves_match_the_restatement(gz, oracle, m, width, max_sweeps):
    rng = np.random.default_rng(m * 100 + width)
    rows, cols = 23, 31
    vol = rng.integers(0, 160, (rows, cols, m)).astype(np.int64)
    p = gz.EnergyParams(int(rng.integers(2, 9)), int(rng.integers(10, 60)))
    lo = rng.integers(0, m - width, (rows, cols)).astype(np.int32)
    hi = np.minimum(lo + width, m - 1).astype(np.int32)
    net = gz.build_network(vol, p, lo=lo, hi=hi)
    r = gz.maxflow_push_relabel(net, max_sweeps=max_sweeps)
    lab, rep = _restated(oracle, vol, p, lo, hi, max_sweeps, r.stats["bfs_h"])
    assert (r.stats["sweeps"], r.stats["pulses"]) == (rep["sweeps"], rep["pulses"])
    assert r.flow == rep["flow"]
    assert np.array_equal(r.labeling, lab)
    assert r.stats["converged"] == bool(rep["converged"])


@pytest.mark.parametrize("max_sweeps", [1, 2, 5])
def test_capped_full_window_m16(gz, oracle, max_sweeps):
    rng = np.random.default_rng(16 + max_sweeps)
    vol = rng.integers(0, 200, (40, 52, 16)).astype(np.int64)
    p = gz.EnergyParams(7, 60)
    r = gz.maxflow_push_relabel(gz.build_network(vol, p), max_sweeps=max_sweeps)
    lo, hi = np.zeros((40, 52), np.int32), np.full((40, 52), 15, np.int32)
    lab, rep = _restated(oracle, vol, p, lo, hi, max_sweeps, r.stats["bfs_h"])
    assert r.flow == rep["flow"] and np.array_equal(r.labeling, lab)


@pytest.mark.parametrize("block", [2, 3])
def test_level2_fine_solve_matches_the_restatement(gz, oracle, block):
    """solve_level2 (hierarchy.py:120-165) on the 24-label Tsukuba-shaped
    ladder scene: the coarse solve and the skin are canonical, the capped fine
    solve is the restated schedule, bit for bit."""
    sc = gz.make_scene(0, 384, 288, 10, 28)
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    p = gz.EnergyParams(14, 1023)
    r = gz.solve_level2(vol, p, block=block)
    cvol, cp = gz.coarsen(vol, block, p)
    coarse = gz.solve_exact(cvol, cp)
    lo, hi = gz.thin_skin(coarse.labeling, vol.shape, block, 1)
    lab, rep = _restated(oracle, vol, p, lo, hi, 8, r.stats["bfs_h"])
    assert np.array_equal(r.labeling, lab)
    assert r.energy == oracle.total_energy(lab, vol, 14, 1023)
    print(f"L2 b={block}: energy {r.energy}, sweeps {rep['sweeps']}, pulses {rep['pulses']}, "
          f"device {r.stats.get('device_ms_total', r.stats['device_ms']):.2f} ms")
