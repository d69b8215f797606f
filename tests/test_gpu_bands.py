"""Row-band solves (gz_solve_volume_banded): one volume split
into bands, one cooperative launch per band, all launches one team.  The cut
is canonical, so every band count must reproduce the one-launch solve and the
reference's fixtures bit for bit.  On a one-GPU box the bands share cuda:0
(devices = (0, 0, ...): each band gets 1/n of the SMs); the placement of band
memory affects speed only, so this exercises the band logic the multi-GPU run
uses: band-local tiles, sites and pulse groups, the cross-launch team barrier,
cross-band arcs and the VMM-mapped workspace."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLDEN / "golden.json").read_text())
BIG = json.loads((GOLDEN / "big.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("nbands", [1, 2, 3, 4])
def test_c1_bands_match_reference(gz, nbands):
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    for seed in (0, 1):
        sc = gz.make_scene(seed)
        vol = gz.sad_volume(sc.left, sc.right, cub)
        r = gz.solve_exact_bands(vol, gz.EnergyParams(14, 1023), devices=(0,) * nbands)
        want = G["c1_exact"][seed]
        assert r.flow == want["flow"] and r.energy == want["energy"], (seed, nbands)
        assert sha(r.labeling) == want["labeling"], (seed, nbands)
        assert r.stats["bands"] == nbands


def test_c2_two_bands_match_reference(gz):
    g = BIG["c2_exact"]
    seed, w, h, dmin, dmax, m = g["args"]
    sc = gz.make_scene(seed, w, h, dmin, dmax)
    cub = gz.cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    r = gz.solve_exact_bands(vol, gz.EnergyParams(14, 1023), devices=(0, 0))
    assert r.flow == g["flow"] and r.energy == g["energy"]
    assert sha(r.labeling.astype(np.int32)) == g["labeling"]
    print("C2 two bands device_ms", r.stats["device_ms"], "sweeps", r.stats["sweeps"])


@pytest.mark.parametrize("m,nbands", [(24, 2), (40, 3), (100, 2), (200, 4)])
def test_random_volumes_bands_equal_one_launch(gz, m, nbands):
    """Multi-segment chains (m > 32) and hard inhibit across band edges."""
    rng = np.random.default_rng(1000 + m)
    rows, cols = 96, 80
    vol = rng.integers(0, 200, size=(rows, cols, m)).astype(np.int64)
    for hard in (False, True):
        p = gz.EnergyParams(9, 40, hard)
        one = gz.solve_exact(vol, p)
        r = gz.solve_exact_bands(vol, p, devices=(0,) * nbands)
        assert r.flow == one.flow and r.energy == one.energy, (m, nbands, hard)
        assert np.array_equal(r.labeling, one.labeling), (m, nbands, hard)


def test_windowed_bands_equal_one_launch(gz):
    """Level-1 style windows (the fine solve of hierarchy.py:92-117)."""
    rng = np.random.default_rng(7)
    rows, cols, m = 120, 100, 24
    vol = rng.integers(0, 300, size=(rows, cols, m)).astype(np.int64)
    center = rng.integers(0, m, size=(rows, cols))
    lo = np.clip(center - 4, 0, m - 1).astype(np.int32)
    hi = np.clip(center + 4, 0, m - 1).astype(np.int32)
    p = gz.EnergyParams(14, 1023)
    net = gz.build_network(vol, p, lo, hi)
    one = gz.maxflow_push_relabel(net)
    r = gz.solve_exact_bands(vol, p, devices=(0, 0), lo=lo, hi=hi)
    assert r.flow == one.flow and r.energy == one.energy
    assert np.array_equal(r.labeling, one.labeling)


def test_band_argument_errors(gz):
    vol = np.zeros((4, 40, 8), np.int64)
    with pytest.raises(ValueError):   # fewer tile rows than bands
        gz.solve_exact_bands(vol, gz.EnergyParams(14, 1023), devices=(0,) * 16)
    with pytest.raises(ValueError):
        gz.solve_exact_bands(vol, gz.EnergyParams(14, 1023), devices=(99,))


@pytest.mark.parametrize("m", [16, 40])
def test_band_worklists_forced(gz, monkeypatch, m):
    """Band-routed pulse worklists (GZ_WORKLIST=1; auto leaves them off for
    bands): every push goes to the list of the target group's band."""
    rng = np.random.default_rng(500 + m)
    vol = rng.integers(0, 300, size=(160, 200, m)).astype(np.int64)
    p = gz.EnergyParams(14, 60)
    one = gz.solve_exact(vol, p)
    monkeypatch.setenv("GZ_WORKLIST", "1")
    for nb in (1, 3):
        r = gz.solve_exact_bands(vol, p, devices=(0,) * nb)
        assert r.flow == one.flow and np.array_equal(r.labeling, one.labeling), (m, nb)


@pytest.fixture
def force_sys(monkeypatch):
    """GZ_FORCE_SYS=1: the multi-device band path on one GPU -- system-scope
    fences and atomics in the team barrier and on cross-band state, and one
    physical VMM allocation per band."""
    monkeypatch.setenv("GZ_FORCE_SYS", "1")


@pytest.mark.parametrize("nbands", [2, 4])
def test_c1_bands_forced_system_scope(gz, force_sys, nbands):
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    for seed in (0, 3):
        sc = gz.make_scene(seed)
        vol = gz.sad_volume(sc.left, sc.right, cub)
        r = gz.solve_exact_bands(vol, gz.EnergyParams(14, 1023), devices=(0,) * nbands)
        want = G["c1_exact"][seed]
        assert r.flow == want["flow"] and r.energy == want["energy"], (seed, nbands)
        assert sha(r.labeling) == want["labeling"], (seed, nbands)


@pytest.mark.parametrize("m,nbands", [(40, 2), (100, 4)])
def test_random_bands_forced_system_scope(gz, force_sys, m, nbands):
    rng = np.random.default_rng(2000 + m)
    rows, cols = 96, 80
    vol = rng.integers(0, 200, size=(rows, cols, m)).astype(np.int64)
    for hard in (False, True):
        p = gz.EnergyParams(9, 40, hard)
        one = gz.solve_exact(vol, p)
        r = gz.solve_exact_bands(vol, p, devices=(0,) * nbands)
        assert (r.flow, r.energy) == (one.flow, one.energy), (m, nbands, hard)
        assert np.array_equal(r.labeling, one.labeling), (m, nbands, hard)
