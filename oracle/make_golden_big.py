"""Golden fixtures for the large BASELINE configs, produced by the REFERENCE itself.

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden_big.py

C2 (450x375, 60 labels): the reference solves it exactly (~4-5 min on one
core) -> volume digest, flow, energy, labeling digest.
C3 (1920x1080, 128 labels): the reference cannot solve it (int32 arc ids,
flownet.py:204-207; 89.6 GB CSR), but its sad_volume runs -> volume digest,
used with the optimality certificate (flow == total_energy(labeling)) in
tests/test_gpu_big.py.
Writes tests/golden/big.json.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

import gazecut as R  # noqa: E402
from gazecut.synthetic import make_scene  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    out = {"generator": "oracle/make_golden_big.py", "reference": "/root/reference/pkg (gazecut 0.1.0)"}
    params = R.EnergyParams(14, 1023)
    # C2
    sc = make_scene(0, 450, 375, 11, 59)
    cub = R.cuboid_from_disparity_range(450, 375, 11, 59, num_labels=60)
    vol = R.sad_volume(sc.left, sc.right, cub)
    t = time.perf_counter()
    r = R.solve_exact(vol, params)
    out["c2_exact"] = {"args": [0, 450, 375, 11, 59, 60], "volume": sha(vol), "flow": r.flow, "energy": r.energy,
                       "labeling": sha(r.labeling.astype(np.int32)), "sweeps": r.stats["sweeps"],
                       "ref_wall_s": time.perf_counter() - t}
    print("c2", out["c2_exact"], flush=True)
    # C3 data term only
    sc = make_scene(0, 1920, 1080, 11, 255)
    cub = R.cuboid_from_disparity_range(1920, 1080, 11, 255, num_labels=128)
    t = time.perf_counter()
    vol = R.sad_volume(sc.left, sc.right, cub)
    out["c3_volume"] = {"args": [0, 1920, 1080, 11, 255, 128], "volume": sha(vol), "shape": list(vol.shape),
                        "ref_wall_s": time.perf_counter() - t}
    print("c3", out["c3_volume"], flush=True)
    (ROOT / "tests" / "golden" / "big.json").write_text(json.dumps(out, indent=1, default=int) + "\n")


if __name__ == "__main__":
    main()
