"""Fixtures for the device accuracy path (ground truth, error counts, penalty
sweeps), produced by running the REFERENCE package itself in this container:

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden_eval.py

-> tests/golden/eval.json.  Inputs are regenerated from seeds by the tests."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

from gazecut.energy import EnergyParams, sad_volume  # noqa: E402
from gazecut.evalreport import error_count, sweep_penalty  # noqa: E402
from gazecut.geometry import cuboid_from_disparity_range  # noqa: E402
from gazecut.imaging import GroundTruthDepth, ground_truth_to_depth  # noqa: E402
from gazecut.maxflow import solve_exact  # noqa: E402
from gazecut.synthetic import make_scene  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gt_record(seed, w, h, dmin, dmax, m):
    sc = make_scene(seed, width=w, height=h, dis_min=dmin, dis_max=dmax)
    cub = cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
    gt = ground_truth_to_depth(sc.gt_image, sc.gt_scale, cub)
    return sc, cub, gt, {
        "args": [seed, w, h, dmin, dmax, m], "depth": sha(gt.depth.astype(np.int32)),
        "valid": sha(gt.valid.astype(np.uint8)), "out_of_range": gt.out_of_range, "off_grid": gt.off_grid,
        "collisions": gt.collisions, "num_valid": gt.num_valid,
    }


def report(rep):
    return {"total_error": rep.total_error, "evaluated": rep.evaluated, "histogram": rep.histogram.tolist()}


out = {"ground_truth": [], "c1_exact_error": None, "sweeps": []}
# ground truth -> depth numbers: C1 seeds 0, 1 and a narrow cuboid (out-of-range pixels)
for args in ((0, 384, 288, 10, 28, 16), (1, 384, 288, 10, 28, 16), (2, 384, 288, 10, 28, 8)):
    out["ground_truth"].append(gt_record(*args)[3])
# error count of the reference's own exact C1 labeling (seed 0)
sc, cub, gt, _ = gt_record(0, 384, 288, 10, 28, 16)
vol = sad_volume(sc.left, sc.right, cub)
res = solve_exact(vol, EnergyParams(14, 1023))
out["c1_exact_error"] = {"labeling": sha(res.labeling.astype(np.int32)), **report(error_count(res.labeling, gt))}
# disparity images (imaging.py:211-246): the C1 exact labeling, and a random labeling at an explicit scale
import tempfile  # noqa: E402
from gazecut.imaging import write_disparity_image  # noqa: E402
with tempfile.TemporaryDirectory() as td:
    p = Path(td) / "d.pgm"
    scale = write_disparity_image(res.labeling, cub, p, 384, 288, comments=("gazecut exact", "penalty 14"))
    out["disparity_images"] = [{"case": "c1_exact", "scale": scale, "sha": sha(np.frombuffer(p.read_bytes(), np.uint8))}]
    c = cuboid_from_disparity_range(64, 12, 3, 13)
    lab = np.random.default_rng(2).integers(0, c.num_labels, c.site_shape).astype(np.int32)
    scale = write_disparity_image(lab, c, p, 64, 12, scale=7)
    out["disparity_images"].append({"case": "random64x12", "scale": scale,
                                    "sha": sha(np.frombuffer(p.read_bytes(), np.uint8))})
# penalty sweeps: a small synthetic scene, and the reference test's random scene (test_evalreport.py:95-101)
sc, cub, gt, _ = gt_record(3, 96, 64, 2, 13, 8)
vol = sad_volume(sc.left, sc.right, cub)
recs = sweep_penalty(vol, gt, [2, 4, 8, 14, 20, 30], inhibit=1023)
out["sweeps"].append({"scene": [3, 96, 64, 2, 13, 8], "inhibit": 1023, "hard": False,
                      "records": [[r.penalty, r.energy, r.flow, r.error, r.exact_fraction] for r in recs]})
recs = sweep_penalty(vol, gt, [4, 14], inhibit=1023, hard_inhibit=True)
out["sweeps"].append({"scene": [3, 96, 64, 2, 13, 8], "inhibit": 1023, "hard": True,
                      "records": [[r.penalty, r.energy, r.flow, r.error, r.exact_fraction] for r in recs]})
rng = np.random.default_rng(52)
rvol = rng.integers(0, 200, (5, 6, 6)).astype(np.int64)
depth = rng.integers(0, 6, (5, 6)).astype(np.int32)
valid = rng.random((5, 6)) < 0.9
recs = sweep_penalty(rvol, GroundTruthDepth(depth=depth, valid=valid), [2, 4, 8], inhibit=50)
out["sweeps"].append({"random_seed": 52, "inhibit": 50, "hard": False,
                      "records": [[r.penalty, r.energy, r.flow, r.error, r.exact_fraction] for r in recs]})
(ROOT / "tests" / "golden" / "eval.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out)[:2000])
