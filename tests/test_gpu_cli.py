"""The thin `solve` CLI (paper_1803_01516_b200/cli.py) against the
reference's own `gazecut solve` outputs for the same synthetic pair
(pkg/tests/test_cli.py:12-132; digests from oracle/make_golden_cli.py):
byte-identical disparity image, labeling dump and stats file, and the
reference's exit codes."""

import hashlib
import json
import os
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "cli.json").read_text())


@pytest.fixture
def pair_dir(tmp_path, gz):
    from paper_1803_01516_b200.imaging import write_pgm, write_ppm
    seed, w, h, dmin, dmax = GOLD["scene"]
    s = gz.make_scene(seed, w, h, dmin, dmax)
    write_ppm(tmp_path / "left.ppm", s.left)
    write_ppm(tmp_path / "right.ppm", s.right)
    write_pgm(tmp_path / "gt.pgm", s.gt_image)
    for n, want in GOLD["inputs"].items():
        assert hashlib.sha256((tmp_path / n).read_bytes()).hexdigest() == want, n
    cwd = os.getcwd()
    os.chdir(tmp_path)
    yield tmp_path
    os.chdir(cwd)


@pytest.mark.parametrize("name", sorted(GOLD["runs"]))
def test_solve_outputs_are_byte_identical_to_the_reference(pair_dir, name):
    from paper_1803_01516_b200.cli import main
    run = GOLD["runs"][name]
    assert main(["solve", "--left", "left.ppm", "--right", "right.ppm", "--out", name, *run["args"]]) == run["rc"]
    for suf, want in run["files"].items():
        got = (pair_dir / (name + suf)).read_bytes()
        assert hashlib.sha256(got).hexdigest() == want, (name, suf, got.decode(errors="replace")[-400:])


def test_exit_codes(pair_dir, capsys):
    """cli.py:48-50, 479-492: usage 2, unreadable / malformed input 3."""
    from paper_1803_01516_b200.cli import main
    assert main(["solve", "--left", "left.ppm", "--right", "right.ppm", "--out", "x"]) == 2   # no range, no gt
    assert "dis-min" in capsys.readouterr().err
    assert main(["solve", "--left", "no.ppm", "--right", "no.ppm", "--dis-min", "3", "--dis-max", "9",
                 "--out", "y"]) == 3
    (pair_dir / "bad.ppm").write_bytes(b"P6\n4 4\n255\nshort")
    assert main(["solve", "--left", "bad.ppm", "--right", "bad.ppm", "--dis-min", "3", "--dis-max", "9",
                 "--out", "z"]) == 3
    assert main(["solve", "--left", "left.ppm", "--right", "right.ppm", "--dis-min", "3", "--dis-max", "11",
                 "--threads", "0", "--out", "t"]) == 2
