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
