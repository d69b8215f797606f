"""Generate tests/golden/c3_crops.json: exact solves of crops of the C3 volume
(1920x1080, 128 labels; the full graph is beyond the reference) by the
REFERENCE package itself (sad_volume + solve_exact, maxflow.py:481-510), so
the device solve of the same crops can be checked bit for bit.

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden_c3crops.py
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, "/root/reference/pkg/src")

import gazecut as R  # noqa: E402
from gazecut.synthetic import make_scene  # noqa: E402

CROPS = [(0, 0, 64, 128), (500, 900, 64, 128), (1016, 1779, 64, 128)]   # (row0, col0, rows, cols)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    args = (0, 1920, 1080, 11, 255, 128)
    seed, w, h, dmin, dmax, m = args
    sc = make_scene(seed, w, h, dmin, dmax)
    cub = R.cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
    vol = R.sad_volume(sc.left, sc.right, cub)
    out = {"generator": "oracle/make_golden_c3crops.py", "reference": "/root/reference/pkg (gazecut 0.1.0)",
           "args": list(args), "crops": []}
    for r0, c0, hh, ww in CROPS:
        crop = np.ascontiguousarray(vol[r0:r0 + hh, c0:c0 + ww])
        t = time.perf_counter()
        r = R.solve_exact(crop, R.EnergyParams(14, 1023))
        print((r0, c0, hh, ww), "flow", r.flow, f"{time.perf_counter() - t:.1f} s", flush=True)
        out["crops"].append({"crop": [r0, c0, hh, ww], "volume": sha(crop), "flow": int(r.flow),
                             "energy": int(r.energy), "labeling": sha(r.labeling.astype(np.int32))})
    (GOLDEN / "c3_crops.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
