"""Host file formats either side of the path (imaging.py:24-125, 262-287 of the
reference): netpbm readers/writers and labeling dumps, with the reference's own
cases (pkg/tests/test_imaging.py).  CPU only."""

import numpy as np
import pytest

from paper_1803_01516_b200.geometry import cuboid_from_disparity_range
from paper_1803_01516_b200.imaging import (
    FileFormatError,
    disparity_of_labeling,
    load_pgm,
    load_ppm,
    read_labeling,
    write_labeling,
    write_pgm,
    write_ppm,
)


def test_round_trips(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (17, 23, 3)).astype(np.uint8)
    write_ppm(tmp_path / "a.ppm", img, comments=("hello", "world"))
    assert np.array_equal(load_ppm(tmp_path / "a.ppm"), img)
    assert (tmp_path / "a.ppm").read_bytes().startswith(b"P6\n# hello\n# world\n23 17\n255\n")
    g = rng.integers(0, 256, (9, 31)).astype(np.uint8)
    write_pgm(tmp_path / "a.pgm", g)
    assert np.array_equal(load_pgm(tmp_path / "a.pgm"), g)


def test_ascii_and_comments(tmp_path):
    p = tmp_path / "a.ppm"
    p.write_bytes(b"P3\n# a comment\n2 1\n# another\n255\n1 2 3  4 5 6\n")
    assert load_ppm(p).tolist() == [[[1, 2, 3], [4, 5, 6]]]
    p = tmp_path / "a.pgm"
    p.write_bytes(b"P2\n3 2\n255\n0 10 20 30 40 50\n")
    assert load_pgm(p)[1, 2] == 50
    img = np.arange(6, dtype=np.uint8).reshape(2, 3)
    p.write_bytes(b"P5 #inline\n3 2 255\n" + img.tobytes())
    assert np.array_equal(load_pgm(p), img)


def test_malformed(tmp_path):
    p = tmp_path / "bad"
    for raw in (b"P7\n1 1\n255\n\x00", b"P5\n4 4\n255\nxy", b"P5\n2 2\n65535\n\x00\x00\x00\x00",
                b"P6\n2 2\n255\n" + bytes(12), b"P5\n2", b"P2\n2 1\n255\n1 300\n"):
        p.write_bytes(raw)
        with pytest.raises(FileFormatError):
            load_pgm(p)
    with pytest.raises(FileNotFoundError):
        load_pgm(tmp_path / "missing.pgm")
    with pytest.raises(ValueError):
        write_pgm(tmp_path / "x.pgm", np.zeros((2, 2), np.int32))


def test_labeling_dump(tmp_path):
    lab = np.random.default_rng(3).integers(-1, 30, (7, 11)).astype(np.int32)
    write_labeling(tmp_path / "l.txt", lab, comments=("config a", "config b"))
    assert np.array_equal(read_labeling(tmp_path / "l.txt"), lab)
    (tmp_path / "bad.txt").write_text("rows 2 wrong 2\n1 2\n3 4\n")
    with pytest.raises(FileFormatError):
        read_labeling(tmp_path / "bad.txt")


def test_disparity_of_labeling():
    c = cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
    lab = np.zeros(c.site_shape, dtype=np.int32)
    assert (disparity_of_labeling(lab, c) == 383 - 2 * c.d_min).all()
    lab[:] = c.num_labels - 1
    assert (disparity_of_labeling(lab, c) == 383 - 2 * c.d_max).all()


def test_csv_writers(tmp_path):
    """evalreport.py:197-233 formats (pkg/tests/test_evalreport.py:120-175)."""
    import csv
    import io

    from paper_1803_01516_b200.evalreport import MethodRow, SweepRecord, write_compare_csv, write_sweep_csv
    recs = [SweepRecord(3, 100, 90, 7, 0.5, 0.25), SweepRecord(6, 120, 110, 5, 0.75, 0.5)]
    write_sweep_csv(tmp_path / "s.csv", recs, comments=("inhibit 30",), timings=True)
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert lines[0] == "# inhibit 30" and lines[1] == "penalty,energy,flow,error,exact_fraction,wall_s"
    assert lines[2] == "3,100,90,7,0.500000,0.250"
    buf = io.StringIO()
    write_sweep_csv(buf, recs[:1], comments=("stream",))
    assert buf.getvalue().splitlines() == ["# stream", "penalty,energy,flow,error,exact_fraction", "3,100,90,7,0.500000"]
    rows = [MethodRow(0, 1, 50, 4, 0.25, 1.0, 30), MethodRow(2, 2, 55, None, None, 2.0, 12, False)]
    write_compare_csv(tmp_path / "c.csv", rows, comments=("a", "b"))
    lines = (tmp_path / "c.csv").read_text().splitlines()
    assert lines[:2] == ["# a", "# b"]
    parsed = list(csv.DictReader(lines[2:]))
    assert parsed[0] == {"level": "0", "block": "1", "energy": "50", "error": "4", "exact_fraction": "0.250000",
                         "nodes": "30", "converged": "1"}
    assert parsed[1]["error"] == "" and parsed[1]["converged"] == "0"
