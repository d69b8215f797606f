"""C5 (3840x2160, 256 labels) data-term digest produced by the REFERENCE's
sad_volume (the reference cannot build the C5 graph).  Adds "c5_volume" to
tests/golden/big.json.

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden_c5.py
"""
import hashlib, json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
import gazecut as R  # noqa: E402
from gazecut.synthetic import make_scene  # noqa: E402

args = [0, 3840, 2160, 11, 511, 256]
sc = make_scene(*args[:5])
cub = R.cuboid_from_disparity_range(*args[1:5], num_labels=args[5])
t = time.perf_counter()
vol = R.sad_volume(sc.left, sc.right, cub)
entry = {"args": args, "volume": hashlib.sha256(np.ascontiguousarray(vol).tobytes()).hexdigest(),
         "shape": list(vol.shape), "ref_wall_s": time.perf_counter() - t}
path = ROOT / "tests" / "golden" / "big.json"
big = json.loads(path.read_text())
big["c5_volume"] = entry
path.write_text(json.dumps(big, indent=1, default=int) + "\n")
print(entry)
