"""Generate tests/golden/ fixtures by running the REFERENCE package itself.

Needs /root/reference (read-only mount, this container only) and numba:

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden.py

The fixtures are small (inputs are regenerated from seeds; outputs are
flows/energies and sha256 digests of labelings / volumes / images), so the
parity tests can run on the GPU box where /root/reference does not exist.
"""

from __future__ import annotations

import hashlib
import io
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, "/root/reference/pkg/src")

import gazecut as R  # noqa: E402
from gazecut.flownet import dump_network  # noqa: E402
from gazecut.synthetic import make_scene  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_cases(seed: int, n: int):
    """Random volumes / params / windows covering the reference test families
    (test_maxflow.py:282-390, test_flownet.py:111-158, test_acceptance.py:259-349)."""
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        rows, cols, m = int(rng.integers(1, 7)), int(rng.integers(1, 7)), int(rng.integers(2, 8))
        vol = rng.integers(0, 200, (rows, cols, m)).astype(np.int64)
        params = R.EnergyParams(penalty=int(rng.integers(0, 9)), inhibit=int(rng.integers(0, 80)),
                                hard_inhibit=bool(rng.integers(5) == 0))
        lo = hi = None
        if i % 3 == 2:
            lo = rng.integers(0, m, rows * cols).astype(np.int32)
            hi = np.minimum(lo + rng.integers(0, m, rows * cols), m - 1).astype(np.int32)
        cases.append((vol, params, lo, hi))
    return cases


def main() -> None:
    GOLDEN.mkdir(parents=True, exist_ok=True)
    out: dict = {"generator": "oracle/make_golden.py", "reference": "/root/reference/pkg (gazecut 0.1.0)"}

    # 1. the reference's own golden arc dump (pkg/tests/test_flownet.py:28-61)
    buf = io.StringIO()
    dump_network(R.build_network(np.array([[[5, 7, 9], [6, 8, 10]]], np.int64), R.EnergyParams(3, 11)), buf)
    out["golden_1x2x3_dump"] = buf.getvalue()

    # 2. synthetic scenes + cuboids
    scenes = {}
    for key, args in {"c1_s0": (0, 384, 288, 10, 28), "c1_s5": (5, 384, 288, 10, 28),
                      "c2_s0": (0, 450, 375, 11, 59), "small_s3": (3, 64, 32, 2, 9)}.items():
        sc = make_scene(*args)
        scenes[key] = {"args": list(args), "left": sha(sc.left), "right": sha(sc.right),
                       "gt": sha(sc.gt_image), "disparity": sha(sc.disparity)}
    out["scenes"] = scenes
    cubs = {}
    for args in [(384, 288, 10, 28, 0, 16), (384, 288, 10, 28, 0, 24), (450, 375, 11, 59, 0, 60),
                 (1920, 1080, 11, 255, 0, 128), (3840, 2160, 11, 511, 0, 256), (64, 32, 2, 9, 0, 6)]:
        c = R.cuboid_from_disparity_range(*args[:5], num_labels=args[5])
        cubs[",".join(map(str, args))] = c.__dict__
    out["cuboids"] = cubs

    # 3. exact solves of the C1 configuration, seeds 0..7 (BASELINE config 1)
    params = R.EnergyParams(14, 1023)
    c1 = []
    cub16 = R.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
    for seed in range(8):
        sc = make_scene(seed)
        vol = R.sad_volume(sc.left, sc.right, cub16)
        t = time.perf_counter()
        r = R.solve_exact(vol, params)
        c1.append({"seed": seed, "volume": sha(vol), "flow": r.flow, "energy": r.energy,
                   "labeling": sha(r.labeling.astype(np.int32)), "sweeps": r.stats["sweeps"],
                   "ref_wall_s": time.perf_counter() - t})
        print("c1 seed", seed, r.flow, flush=True)
    out["c1_exact"] = c1

    # 4. the 24-label acceptance scene: exact + hierarchy ladder (pkg/test_output.txt:24)
    cub24 = R.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
    sc = make_scene(0)
    vol24 = R.sad_volume(sc.left, sc.right, cub24)
    ladder = {"volume": sha(vol24)}
    ex = R.solve_exact(vol24, params)
    ladder["exact"] = {"flow": ex.flow, "energy": ex.energy, "labeling": sha(ex.labeling.astype(np.int32))}
    for name, fn in (("l1b2", lambda: R.solve_level1(vol24, params, 2)),
                     ("l1b3", lambda: R.solve_level1(vol24, params, 3)),
                     ("l2b3", lambda: R.solve_level2(vol24, params, 3))):
        r = fn()
        ladder[name] = {"energy": r.energy, "labeling": sha(r.labeling.astype(np.int32)),
                        "coarse_energy": r.stats["coarse_energy"], "converged": bool(r.stats["converged"])}
        print("ladder", name, r.energy, flush=True)
    out["ladder24"] = ladder

    # 5. level-1 on C1 (16 labels), b = 2 and 4
    sc = make_scene(0)
    vol16 = R.sad_volume(sc.left, sc.right, cub16)
    out["c1_level1"] = {}
    for b in (2, 4):
        r = R.solve_level1(vol16, params, b)
        out["c1_level1"][str(b)] = {"energy": r.energy, "flow": r.flow, "labeling": sha(r.labeling.astype(np.int32)),
                                    "coarse_energy": r.stats["coarse_energy"]}

    # 6. random small cases with full inputs/outputs
    cases = random_cases(2031, 90)
    arrays = {}
    meta = []
    for i, (vol, p, lo, hi) in enumerate(cases):
        net = R.build_network(vol, p, lo, hi)
        r = R.maxflow_push_relabel(net)
        arrays[f"vol{i}"] = vol
        arrays[f"lab{i}"] = r.labeling.astype(np.int32)
        arrays[f"side{i}"] = r.source_side
        if lo is not None:
            arrays[f"lo{i}"] = lo
            arrays[f"hi{i}"] = hi
        meta.append({"penalty": p.penalty, "inhibit": p.inhibit, "hard": p.hard_inhibit, "windowed": lo is not None,
                     "flow": r.flow, "energy": r.energy, "const_offset": net.const_offset,
                     "nodes": net.n_nodes, "arcs": net.num_arcs,
                     "total_energy": int(R.total_energy(r.labeling, vol, p))})
    np.savez_compressed(GOLDEN / "random_cases.npz", **arrays)
    out["random_cases"] = meta

    # 7. hierarchy on random volumes (test_hierarchy.py:52-107 families)
    rng = np.random.default_rng(2032)
    hier = []
    harr = {}
    for i in range(12):
        vol = rng.integers(0, 300, (int(rng.integers(4, 11)), int(rng.integers(4, 11)), int(rng.integers(4, 12)))).astype(np.int64)
        p = R.EnergyParams(penalty=int(rng.integers(1, 9)), inhibit=int(rng.integers(0, 90)))
        b = int(rng.integers(1, 4))
        c, cp = R.coarsen(vol, b, p)
        l1 = R.solve_level1(vol, p, b)
        l2u = R.solve_level2(vol, p, b, max_sweeps=None)
        harr[f"vol{i}"] = vol
        harr[f"coarse{i}"] = c
        harr[f"l1lab{i}"] = l1.labeling.astype(np.int32)
        hier.append({"penalty": p.penalty, "inhibit": p.inhibit, "block": b, "coarse_penalty": cp.penalty,
                     "l1_energy": l1.energy, "l1_flow": l1.flow, "coarse_energy": l1.stats["coarse_energy"],
                     "l2u_energy": l2u.energy, "l2u_same_as_l1": bool(np.array_equal(l2u.labeling, l1.labeling))})
    np.savez_compressed(GOLDEN / "hierarchy_cases.npz", **harr)
    out["hierarchy_cases"] = hier

    (GOLDEN / "golden.json").write_text(json.dumps(out, indent=1, default=int) + "\n")
    print("wrote", GOLDEN)


if __name__ == "__main__":
    main()
