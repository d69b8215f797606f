"""Host-side pieces that need no GPU: geometry, synthetic scenes, graph-size model."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1803_01516_b200 as gz
from paper_1803_01516_b200.flownet import graph_size

G = json.loads((Path(__file__).resolve().parent / "golden" / "golden.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("key", list(G["scenes"]))
def test_scenes_match_reference(key):
    want = G["scenes"][key]
    sc = gz.make_scene(*want["args"])
    assert sha(sc.left) == want["left"] and sha(sc.right) == want["right"]
    assert sha(sc.gt_image) == want["gt"] and sha(sc.disparity) == want["disparity"]


@pytest.mark.parametrize("key", list(G["cuboids"]))
def test_cuboids_match_reference(key):
    a = [int(x) for x in key.split(",")]
    c = gz.cuboid_from_disparity_range(*a[:5], num_labels=a[5])
    assert c.__dict__ == G["cuboids"][key]


def test_tsukuba_cuboid_frozen():
    # pkg/tests/test_geometry.py:94-103 family: 384x288, dis 10..28, 24 labels
    c = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
    assert (c.g_extent, c.y_extent, c.num_labels) == (372, 288, 24)
    assert gz.expected_node_count(c.site_shape, 24) == 2_464_130
    assert gz.expected_arc_count(c.site_shape, 24) == 33_766_536


def test_graph_size_model_matches_reference_counts():
    arr = np.load(Path(__file__).resolve().parent / "golden" / "random_cases.npz")
    for i, meta in enumerate(G["random_cases"]):
        vol = torch.from_numpy(arr[f"vol{i}"].astype(np.int32))
        p = gz.EnergyParams(meta["penalty"], meta["inhibit"], meta["hard"])
        lo = torch.from_numpy(arr[f"lo{i}"]) if meta["windowed"] else None
        hi = torch.from_numpy(arr[f"hi{i}"]) if meta["windowed"] else None
        assert graph_size(vol, p, lo, hi) == (meta["nodes"], meta["arcs"], meta["const_offset"]), i


def test_round_trips_small_widths():
    # pkg/tests/test_acceptance.py:308-331 (criterion 6d), widths 2..40
    for w in range(2, 41):
        for d in range((w + 1) // 2):
            for g in range(-d, w - d):
                if not 0 <= (w - 1) + g - d < w:
                    continue
                xl, xr, _ = gz.pixels_from_gaze_depth((g, d, 0), w)
                cr = gz.cross_from_pixels(xl, xr, 0, w)
                assert cr is not None and (cr.g, cr.d) == (g, d)


def test_pairwise_table():
    p = gz.EnergyParams(14, 1023)
    assert [gz.pairwise_term(4, j, p) for j in (4, 5, 6)] == [0, 14, 2 * 14 + 1023]
    assert gz.pairwise_term(0, 5, p) == 5 * 14 + 4 * 1023
    with pytest.raises(ValueError):
        gz.EnergyParams(-1, 3)
