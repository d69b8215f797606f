"""Generate tests/golden/cli.json: the reference CLI's output files
(`gazecut solve`, cli.py:179-249) for the synthetic 64x32 pair of
pkg/tests/test_cli.py:12-20, as sha256 digests, by running the REFERENCE
itself here (relative file names, so the header comments are path-free).

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/make_golden_cli.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")

from gazecut.cli import main  # noqa: E402
from gazecut.imaging import write_pgm, write_ppm  # noqa: E402
from gazecut.synthetic import make_scene  # noqa: E402

RUNS = {
    "exact": ["--dis-min", "3", "--dis-max", "11"],
    "exact_gt": ["--gt", "gt.pgm"],
    "level1_b2": ["--dis-min", "3", "--dis-max", "11", "--level", "1", "--block", "2", "--gt", "gt.pgm"],
    "level2_b2": ["--dis-min", "3", "--dis-max", "11", "--level", "2", "--block", "2"],
    "hard_scale4": ["--dis-min", "3", "--dis-max", "11", "--hard-inhibit", "--scale", "4"],
}


def main_() -> None:
    out = {"generator": "oracle/make_golden_cli.py", "scene": [3, 64, 32, 3, 11], "runs": {}}
    cwd = os.getcwd()
    with tempfile.TemporaryDirectory() as d:
        os.chdir(d)
        s = make_scene(seed=3, width=64, height=32, dis_min=3, dis_max=11)
        write_ppm("left.ppm", s.left)
        write_ppm("right.ppm", s.right)
        write_pgm("gt.pgm", s.gt_image)
        out["inputs"] = {n: hashlib.sha256(Path(n).read_bytes()).hexdigest() for n in ("left.ppm", "right.ppm", "gt.pgm")}
        for name, extra in RUNS.items():
            rc = main(["solve", "--left", "left.ppm", "--right", "right.ppm", "--out", name, *extra])
            files = {suf: hashlib.sha256(Path(name + suf).read_bytes()).hexdigest()
                     for suf in (".pgm", ".labels.txt", ".stats.txt")}
            out["runs"][name] = {"args": extra, "rc": rc, "files": files,
                                 "stats": Path(name + ".stats.txt").read_text()}
        os.chdir(cwd)
    (ROOT / "tests" / "golden" / "cli.json").write_text(json.dumps(out, indent=1))
    print("wrote tests/golden/cli.json")


if __name__ == "__main__":
    main_()
