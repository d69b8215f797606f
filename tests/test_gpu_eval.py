"""Device accuracy accounting and penalty sweeps
against fixtures produced by running the reference (tests/golden/eval.json,
oracle/make_golden_eval.py) and against the numpy oracle on random inputs."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
E = json.loads((GOLDEN / "eval.json").read_text())
G = json.loads((GOLDEN / "golden.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _scene_gt(gz, seed, w, h, dmin, dmax, m):
    sc = gz.make_scene(seed, w, h, dmin, dmax)
    cub = gz.cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
    return sc, cub, gz.ground_truth_to_depth(sc.gt_image, sc.gt_scale, cub)


def test_ground_truth_to_depth_matches_reference(gz):
    for g in E["ground_truth"]:
        _, _, gt = _scene_gt(gz, *g["args"])
        assert sha(gt.depth.astype(np.int32)) == g["depth"], g["args"]
        assert sha(gt.valid.astype(np.uint8)) == g["valid"], g["args"]
        assert (gt.out_of_range, gt.off_grid, gt.collisions, gt.num_valid) == \
            (g["out_of_range"], g["off_grid"], g["collisions"], g["num_valid"])


def test_ground_truth_random_vs_oracle(gz, oracle):
    rng = np.random.default_rng(77)
    cub = gz.cuboid_from_disparity_range(120, 40, 3, 21, num_labels=7)
    img = rng.integers(0, 256, (40, 120)).astype(np.uint8)
    img[rng.random(img.shape) < 0.3] = 0
    for scale in (1, 3, 8):
        gt = gz.ground_truth_to_depth(img, scale, cub)
        d, v, oor, off, coll = oracle.ground_truth_to_depth(
            img, scale, cub.g_min, cub.y_min, cub.d_min, cub.y_extent, cub.g_extent, cub.num_labels, cub.offset1,
            cub.offset2, cub.offset3, cub.lw_offset, cub.rw_offset, cub.h_offset)
        assert np.array_equal(gt.depth, d) and np.array_equal(gt.valid, v)
        assert (gt.out_of_range, gt.off_grid, gt.collisions) == (oor, off, coll)


def test_error_count_reference_cases(gz):
    gt = gz.GroundTruthDepth(depth=np.array([[3, 5, 0], [2, 2, 9]], np.int32),
                             valid=np.array([[True, True, False], [True, True, True]]))
    rep = gz.error_count(np.array([[3, 7, 4], [1, 2, 20]]), gt)
    assert rep.total_error == 14 and rep.evaluated == 5
    assert list(rep.histogram[:3]) == [2, 1, 1] and rep.histogram[9] == 1
    assert rep.exact_fraction == pytest.approx(2 / 5)
    assert rep.rows()[0] == ("0", 2) and rep.rows()[-1] == ("9~", 1)
    with pytest.raises(ValueError):
        gz.error_count(np.zeros((2, 2)), gz.GroundTruthDepth(depth=np.zeros((1, 1), np.int32),
                                                             valid=np.ones((1, 1), bool)))


def test_error_count_random_vs_oracle(gz, oracle):
    rng = np.random.default_rng(57)
    depth = rng.integers(0, 40, (97, 131)).astype(np.int32)
    valid = rng.random(depth.shape) < 0.7
    gt = gz.GroundTruthDepth(depth=depth, valid=valid)
    for tail in (1, 9, 30):
        lab = rng.integers(0, 40, depth.shape).astype(np.int32)
        rep = gz.error_count(lab, gt, tail)
        tot, ev, hist = oracle.error_count(lab, depth, valid, tail)
        assert (rep.total_error, rep.evaluated) == (tot, ev) and np.array_equal(rep.histogram, hist)
    assert gz.error_count(depth, gt).total_error == 0


def test_c1_exact_error_matches_reference(gz):
    sc, cub, gt = _scene_gt(gz, 0, 384, 288, 10, 28, 16)
    r = gz.solve_exact(gz.sad_volume(sc.left, sc.right, cub), gz.EnergyParams(14, 1023))
    want = E["c1_exact_error"]
    assert sha(r.labeling.astype(np.int32)) == want["labeling"] == G["c1_exact"][0]["labeling"]
    rep = gz.error_count(r.labeling, gt)
    assert (rep.total_error, rep.evaluated, rep.histogram.tolist()) == \
        (want["total_error"], want["evaluated"], want["histogram"])


def test_sweep_penalty_matches_reference(gz):
    for sw in E["sweeps"]:
        if "scene" in sw:
            sc, cub, gt = _scene_gt(gz, *sw["scene"])
            vol = gz.sad_volume(sc.left, sc.right, cub)
        else:
            rng = np.random.default_rng(sw["random_seed"])
            vol = rng.integers(0, 200, (5, 6, 6)).astype(np.int64)
            depth = rng.integers(0, 6, (5, 6)).astype(np.int32)
            valid = rng.random((5, 6)) < 0.9
            gt = gz.GroundTruthDepth(depth=depth, valid=valid)
        pens = [r[0] for r in sw["records"]]
        recs = gz.sweep_penalty(vol, gt, pens, inhibit=sw["inhibit"], hard_inhibit=sw["hard"])
        got = [[r.penalty, r.energy, r.flow, r.error] for r in recs]
        assert got == [r[:4] for r in sw["records"]], sw.get("scene", sw.get("random_seed"))
        for r, w in zip(recs, sw["records"]):
            assert r.exact_fraction == pytest.approx(w[4], abs=0, rel=1e-12)
        best = gz.best_penalty(recs)
        assert min(r.error for r in recs) == next(r.error for r in recs if r.penalty == best)


def test_sweep_penalty_c1_fifteen_penalties(gz):
    """The paper's Fig. 6 sweep (penalties 2..30 step 2) on C1 seed 0 as one
    batched call; penalty 14 reproduces the reference's exact energy."""
    sc, cub, gt = _scene_gt(gz, 0, 384, 288, 10, 28, 16)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    recs = gz.sweep_penalty(vol, gt, range(2, 31, 2), inhibit=1023)
    by = {r.penalty: r for r in recs}
    assert by[14].energy == G["c1_exact"][0]["energy"] == 778554
    assert by[14].error == E["c1_exact_error"]["total_error"]
    energies = [r.energy for r in recs]
    assert energies == sorted(energies)
    print("C1 sweep best penalty", gz.best_penalty(recs), "wall per solve", recs[0].wall_s)


def test_disparity_images_byte_identical_to_reference(gz, tmp_path):
    """imaging.py:211-246 through the device raster (gz_render_disparity)."""
    want = {d["case"]: d for d in E["disparity_images"]}
    sc, cub, gt = _scene_gt(gz, 0, 384, 288, 10, 28, 16)
    r = gz.solve_exact(gz.sad_volume(sc.left, sc.right, cub), gz.EnergyParams(14, 1023))
    p = tmp_path / "d.pgm"
    scale = gz.write_disparity_image(r.labeling, cub, p, 384, 288, comments=("gazecut exact", "penalty 14"))
    assert scale == want["c1_exact"]["scale"]
    assert sha(np.frombuffer(p.read_bytes(), np.uint8)) == want["c1_exact"]["sha"]
    c = gz.cuboid_from_disparity_range(64, 12, 3, 13)
    lab = np.random.default_rng(2).integers(0, c.num_labels, c.site_shape).astype(np.int32)
    assert gz.write_disparity_image(lab, c, p, 64, 12, scale=7) == 7
    assert sha(np.frombuffer(p.read_bytes(), np.uint8)) == want["random64x12"]["sha"]
    # ground-truth round trip (test_imaging.py:78-94): written image -> depth numbers
    s2 = gz.write_disparity_image(lab, c, p, 64, 12)
    g2 = gz.ground_truth_to_depth(gz.load_pgm(p), s2, c)
    assert g2.num_valid > 0.5 * c.num_sites and g2.out_of_range == 0
    assert np.array_equal(g2.depth[g2.valid], lab[g2.valid])
    with pytest.raises(ValueError):
        gz.write_disparity_image(np.zeros(gz.cuboid_from_disparity_range(64, 4, 1, 31).site_shape, np.int32),
                                 gz.cuboid_from_disparity_range(64, 4, 1, 31), p, 64, 4, scale=100)


def test_compare_methods_ladder(gz):
    """evalreport.py:148-186 on the 24-label ladder: the reference's recorded
    energies (pkg/test_output.txt:24) for exact / l1b2 / l1b3, e0 <= e1 <= e2."""
    sc, cub, gt = _scene_gt(gz, 0, 384, 288, 10, 28, 24)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    rows = gz.compare_methods(vol, gz.EnergyParams(14, 1023), [(0, 1), (1, 2), (1, 3), (2, 3)], gt=gt)
    assert [r.energy for r in rows[:3]] == [778554, 785090, 790627]
    assert rows[0].energy <= rows[1].energy and rows[2].energy <= rows[3].energy
    assert all(r.error is not None and r.nodes > 0 for r in rows)
    with pytest.raises(ValueError):
        gz.compare_methods(vol, gz.EnergyParams(14, 1023), [(3, 1)])
