"""Pin the CPU oracle (oracle/gz_oracle.c) to the reference: its golden arc dump
(pkg/tests/test_flownet.py:28-61), recorded energies (pkg/test_output.txt:24) and
fixtures produced by running the reference itself (oracle/make_golden.py)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLDEN / "golden.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_golden_dump_1x2x3(oracle):
    net = oracle.build_network(np.array([[[5, 7, 9], [6, 8, 10]]], np.int64), 3, 11)
    assert net.dump() == G["golden_1x2x3_dump"]
    assert net.chain_base.tolist() == [0, 3, 6]
    assert net.cap[net.chain_arcs].tolist() == [5, 7, 9, 6, 8, 10]


def test_random_cases_match_reference(oracle):
    arr = np.load(GOLDEN / "random_cases.npz")
    for i, meta in enumerate(G["random_cases"]):
        vol = arr[f"vol{i}"]
        icap = oracle.UNCUTTABLE if meta["hard"] else meta["inhibit"]
        lo = arr[f"lo{i}"] if meta["windowed"] else None
        hi = arr[f"hi{i}"] if meta["windowed"] else None
        net = oracle.build_network(vol, meta["penalty"], icap, lo, hi)
        assert (net.n_nodes, net.num_arcs, net.const_offset) == (meta["nodes"], meta["arcs"], meta["const_offset"])
        flow, energy, lab, side, _ = oracle.maxflow_push_relabel(net)
        assert flow == meta["flow"] and energy == meta["energy"], i
        assert np.array_equal(lab, arr[f"lab{i}"]) and np.array_equal(side, arr[f"side{i}"]), i
        assert oracle.total_energy(lab, vol, meta["penalty"], meta["inhibit"], meta["hard"]) == meta["total_energy"]


def test_hierarchy_cases_match_reference(oracle):
    arr = np.load(GOLDEN / "hierarchy_cases.npz")
    for i, meta in enumerate(G["hierarchy_cases"]):
        vol = arr[f"vol{i}"]
        c, cp = oracle.coarsen(vol, meta["block"], meta["penalty"])
        assert np.array_equal(c, arr[f"coarse{i}"]) and cp == meta["coarse_penalty"]
        r = oracle.solve_level1(vol, meta["penalty"], meta["inhibit"], meta["block"])
        assert r["energy"] == meta["l1_energy"] and r["flow"] == meta["l1_flow"]
        assert r["coarse_energy"] == meta["coarse_energy"]
        assert np.array_equal(r["labeling"], arr[f"l1lab{i}"])


def test_thin_skin_frozen_values(oracle):
    # pkg/tests/test_hierarchy.py:31-40
    lo, hi = oracle.thin_skin(np.array([[0, 2], [1, 3]]), (4, 4, 12), block=3, radius=1)
    assert (lo[0, 0], hi[0, 0], lo[0, 3], hi[0, 3]) == (0, 5, 3, 11)
    assert (lo[3, 0], hi[3, 0], lo[3, 3], hi[3, 3]) == (0, 8, 6, 11)


def _c1_volume(oracle, seed, m):
    import paper_1803_01516_b200 as gz   # host-side scene + cuboid (pinned in test_host.py)
    sc = gz.make_scene(seed)
    c = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=m)
    return oracle.sad_volume(sc.left, sc.right, c.g_min, c.g_extent, c.y_min, c.y_extent, c.d_min, m)


def test_c1_seed0_exact(oracle):
    vol = _c1_volume(oracle, 0, 16)
    want = G["c1_exact"][0]
    assert sha(vol.astype(np.int64)) == want["volume"]
    r = oracle.solve_exact(vol, 14, 1023)
    assert r["flow"] == want["flow"] == 778554 and r["energy"] == want["energy"]
    assert sha(r["labeling"].astype(np.int32)) == want["labeling"]


def test_ladder24_recorded_energies(oracle):
    """pkg/test_output.txt:24 records 778554 / 785090 / 790627 / 790883."""
    vol = _c1_volume(oracle, 0, 24)
    lad = G["ladder24"]
    assert sha(vol.astype(np.int64)) == lad["volume"]
    l1 = oracle.solve_level1(vol, 14, 1023, 2)
    assert l1["energy"] == lad["l1b2"]["energy"] == 785090
    assert sha(l1["labeling"].astype(np.int32)) == lad["l1b2"]["labeling"]
    l2 = oracle.solve_level2(vol, 14, 1023, 3)
    assert l2["energy"] == lad["l2b3"]["energy"] == 790883
    assert sha(l2["labeling"].astype(np.int32)) == lad["l2b3"]["labeling"]


def test_oracle_accuracy_matches_reference_fixtures():
    """oracle.ground_truth_to_depth / error_count against tests/golden/eval.json
    (produced by the reference itself, oracle/make_golden_eval.py)."""
    import hashlib
    import json
    from pathlib import Path

    from oracle import oracle as o
    from paper_1803_01516_b200.geometry import cuboid_from_disparity_range
    from paper_1803_01516_b200.synthetic import make_scene

    E = json.loads((Path(__file__).resolve().parent / "golden" / "eval.json").read_text())
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for g in E["ground_truth"]:
        seed, w, h, dmin, dmax, m = g["args"]
        sc = make_scene(seed, width=w, height=h, dis_min=dmin, dis_max=dmax)
        c = cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
        depth, valid, oor, off, coll = o.ground_truth_to_depth(
            sc.gt_image, sc.gt_scale, c.g_min, c.y_min, c.d_min, c.y_extent, c.g_extent, m, c.offset1, c.offset2,
            c.offset3, c.lw_offset, c.rw_offset, c.h_offset)
        assert sha(depth) == g["depth"] and sha(valid.astype(np.uint8)) == g["valid"]
        assert (oor, off, coll) == (g["out_of_range"], g["off_grid"], g["collisions"])
    # the reference's hand case (test_evalreport.py:34-47)
    tot, ev, hist = o.error_count([[3, 7, 4], [1, 2, 20]], [[3, 5, 0], [2, 2, 9]],
                                  [[True, True, False], [True, True, True]])
    assert (tot, ev) == (14, 5) and hist[0] == 2 and hist[1] == 1 and hist[2] == 1 and hist[9] == 1
