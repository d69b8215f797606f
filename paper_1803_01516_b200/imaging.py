"""Image formats either side of the path and ground truth on the device
(imaging.py of the reference).

* netpbm I/O (imaging.py:24-125): 8-bit P2/P3/P5/P6 readers, binary P5/P6
  writers with header comments -- host file parsing, byte-identical output;
* ``write_disparity_image`` (imaging.py:211-246): the labeling's disparity
  raster is painted on the device (gz_render_disparity), the file written here;
* ``ground_truth_to_depth`` (imaging.py:155-201) on the device
  (gz_ground_truth_to_depth);
* labeling text dumps (imaging.py:262-287)."""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np
import torch

from . import _dev, _lib
from .geometry import CuboidSpec


class FileFormatError(ValueError):
    """imaging.py:20-21: a file that cannot be parsed as what it claims to be."""


# ---------------------------------------------------------------------------
# netpbm (imaging.py:24-125)



def _header(data: bytes, n: int, pos: int, path) -> tuple[list[bytes], int]:
    """n header tokens from pos; '#' starts a comment that runs to end of line."""
    toks: list[bytes] = []
    end = len(data)
    while len(toks) < n:
        if pos >= end:
            raise FileFormatError(f"{path}: truncated netpbm header")
        ch = data[pos:pos + 1]
        if ch in (b" ", b"\t", b"\n", b"\r", b"\v", b"\f"):
            pos += 1
        elif ch == b"#":
            nl = [i for i in (data.find(b"\n", pos), data.find(b"\r", pos)) if i >= 0]
            pos = min(nl) if nl else end
        else:
            q = pos
            while q < end and data[q:q + 1] not in (b" ", b"\t", b"\n", b"\r", b"\v", b"\f", b"#"):
                q += 1
            toks.append(data[pos:q])
            pos = q
    return toks, pos


def _load_netpbm(path) -> np.ndarray:
    data = Path(path).read_bytes()
    (magic,), pos = _header(data, 1, 0, path)
    kinds = {b"P2": (1, False), b"P3": (3, False), b"P5": (1, True), b"P6": (3, True)}
    if magic not in kinds:
        raise FileFormatError(f"{path}: unsupported netpbm magic {magic!r}")
    channels, binary = kinds[magic]
    toks, pos = _header(data, 3, pos, path)
    try:
        width, height, maxval = (int(t) for t in toks)
    except ValueError:
        raise FileFormatError(f"{path}: bad netpbm header {toks!r}") from None
    if width < 1 or height < 1:
        raise FileFormatError(f"{path}: bad dimensions {width}x{height}")
    if maxval != 255:
        raise FileFormatError(f"{path}: only maxval 255 supported, got {maxval}")
    count = width * height * channels
    if binary:
        body = data[pos + 1:pos + 1 + count]   # exactly one whitespace byte ends the header
        if len(body) < count:
            raise FileFormatError(f"{path}: truncated pixel data ({len(body)}/{count} bytes)")
        px = np.frombuffer(body, dtype=np.uint8).copy()
    else:
        vals = data[pos:].split()
        if len(vals) < count:
            raise FileFormatError(f"{path}: truncated pixel data ({len(vals)}/{count} values)")
        px = np.array([int(v) for v in vals[:count]], dtype=np.int64)
        if px.size and (px.min() < 0 or px.max() > maxval):
            raise FileFormatError(f"{path}: sample outside [0, {maxval}]")
        px = px.astype(np.uint8)
    return px.reshape((height, width, 3) if channels == 3 else (height, width))


def load_ppm(path) -> np.ndarray:
    """8-bit colour image (P3/P6) -> uint8 (h, w, 3)."""
    img = _load_netpbm(path)
    if img.ndim != 3:
        raise FileFormatError(f"{path}: expected a colour image, got greyscale")
    return img


def load_pgm(path) -> np.ndarray:
    """8-bit greyscale image (P2/P5) -> uint8 (h, w)."""
    img = _load_netpbm(path)
    if img.ndim != 2:
        raise FileFormatError(f"{path}: expected a greyscale image, got colour")
    return img


def _write_netpbm(path, img, magic: str, comments) -> None:
    a = np.asarray(img)
    if a.dtype != np.uint8:
        raise ValueError(f"expected uint8 image, got {a.dtype}")
    head = [magic] + [f"# {c}" for c in comments] + [f"{a.shape[1]} {a.shape[0]}", "255"]
    Path(path).write_bytes(("\n".join(head) + "\n").encode("ascii") + np.ascontiguousarray(a).tobytes())


def write_ppm(path, img, comments=()) -> None:
    """uint8 (h, w, 3) -> binary P6."""
    a = np.asarray(img)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"expected (h, w, 3), got {a.shape}")
    _write_netpbm(path, a, "P6", comments)


def write_pgm(path, img, comments=()) -> None:
    """uint8 (h, w) -> binary P5."""
    a = np.asarray(img)
    if a.ndim != 2:
        raise ValueError(f"expected (h, w), got {a.shape}")
    _write_netpbm(path, a, "P5", comments)


@dataclass
class GroundTruthDepth:
    """imaging.py:133-152: per-site depth numbers and validity (site grid)."""

    depth: np.ndarray
    valid: np.ndarray
    out_of_range: int = 0
    off_grid: int = 0
    collisions: int = 0
    depth_dev: Optional[torch.Tensor] = field(default=None, repr=False, compare=False)
    valid_dev: Optional[torch.Tensor] = field(default=None, repr=False, compare=False)

    @property
    def num_valid(self) -> int:
        return int(np.asarray(self.valid).sum())

    def device_arrays(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(depth int32, valid uint8) on the device, uploaded once."""
        if self.depth_dev is None or self.valid_dev is None:
            self.depth_dev = _dev.as_device_i32(self.depth, "ground-truth depth").contiguous()
            self.valid_dev = _dev.as_device_u8(np.asarray(self.valid, dtype=bool).astype(np.uint8))
        return self.depth_dev, self.valid_dev


def gaze_struct(cuboid: CuboidSpec) -> _lib.Gaze:
    return _lib.Gaze(cuboid.g_min, cuboid.y_min, cuboid.d_min, cuboid.y_extent, cuboid.g_extent,
                     cuboid.num_labels, cuboid.offset1, cuboid.offset2, cuboid.offset3,
                     cuboid.lw_offset, cuboid.rw_offset, cuboid.h_offset)


def ground_truth_to_depth(gt_image, scale: int, cuboid: CuboidSpec) -> GroundTruthDepth:
    """imaging.py:155-201: a scaled disparity image (v > 0: disparity
    round(v / scale); 0: none) carried through the cuboid transform to per-site
    depth numbers on the device; the nearer surface wins a collision."""
    gt = np.asarray(gt_image) if not isinstance(gt_image, torch.Tensor) else gt_image
    if gt.ndim != 2:
        raise ValueError("ground truth must be a greyscale image")
    if scale < 1:
        raise ValueError("scale must be >= 1")
    h, w = (int(s) for s in gt.shape)
    cuboid.check_consistent(w, h)
    g = _dev.as_device_u8(gt)
    rows, cols = cuboid.site_shape
    depth = torch.empty((rows, cols), dtype=torch.int32, device=g.device)
    valid = torch.empty((rows, cols), dtype=torch.uint8, device=g.device)
    counts = torch.empty(4, dtype=torch.int64, device=g.device)
    gz = gaze_struct(cuboid)
    import ctypes as C
    rc = _lib.lib().gz_ground_truth_to_depth(_dev.ptr(g), h, w, int(scale), C.byref(gz), _dev.ptr(depth),
                                             _dev.ptr(valid), _dev.ptr(counts), _dev.stream_ptr())
    _lib.check(rc, "gz_ground_truth_to_depth")
    oor, off, kept, nvalid = (int(x) for x in counts.cpu())
    return GroundTruthDepth(depth=depth.cpu().numpy(), valid=valid.cpu().numpy().astype(bool),
                            out_of_range=oor, off_grid=off, collisions=kept - nvalid,
                            depth_dev=depth, valid_dev=valid)


# ---------------------------------------------------------------------------
# labeling -> disparity image (imaging.py:204-246)

def disparity_of_labeling(labeling, cuboid: CuboidSpec) -> np.ndarray:
    """imaging.py:204-208: disparity of each site's label (int64 grid)."""
    d = cuboid.d_min + np.asarray(labeling, dtype=np.int64)
    return (cuboid.lw_offset - cuboid.rw_offset) - 2 * (d + cuboid.offset3)


def render_disparity_device(labeling, cuboid: CuboidSpec, width: int, height: int, scale: int) -> torch.Tensor:
    """The disparity raster of a labeling, painted on the device: uint8 (h, w)."""
    lab = _dev.as_device_i32(labeling, "labeling").contiguous()
    scratch = torch.empty(height * width, dtype=torch.int32, device=lab.device)
    img = torch.empty((height, width), dtype=torch.uint8, device=lab.device)
    gz = gaze_struct(cuboid)
    import ctypes as C
    rc = _lib.lib().gz_render_disparity(_dev.ptr(lab), C.byref(gz), int(width), int(height), int(scale),
                                        _dev.ptr(scratch), _dev.ptr(img), _dev.stream_ptr())
    _lib.check(rc, "gz_render_disparity")
    return img


def write_disparity_image(labeling, cuboid: CuboidSpec, path, width: int, height: int, scale=None,
                          comments=()) -> int:
    """imaging.py:211-246: the labeling as a scaled disparity image over the
    right view (nearer surface wins a shared pixel, uncovered pixels 0); the
    scale (largest that cannot clip when None) goes into a header comment and
    is returned.  An explicit clipping scale raises ValueError."""
    cuboid.check_consistent(width, height)
    shape = tuple(labeling.shape)
    if shape != tuple(cuboid.site_shape):
        raise ValueError(f"labeling shape {shape} != {cuboid.site_shape}")
    dis_max = (width - 1) - 2 * cuboid.d_min
    if scale is None:
        scale = max(1, 255 // max(dis_max, 1))
    if scale * dis_max > 255:
        raise ValueError(f"scale {scale} overflows: max disparity {dis_max} -> {scale * dis_max} > 255")
    img = render_disparity_device(labeling, cuboid, width, height, scale).cpu().numpy()
    write_pgm(path, img, comments=tuple(comments) + (f"disparity scale {scale}",))
    return int(scale)


# ---------------------------------------------------------------------------
# labeling dumps (imaging.py:262-287)

def write_labeling(path, labeling, comments=()) -> None:
    """Text dump: '# ' comments, 'rows R cols C', then one line per row."""
    a = np.asarray(labeling)
    lines = [f"# {c}" for c in comments] + [f"rows {a.shape[0]} cols {a.shape[1]}"]
    lines += [" ".join(str(int(v)) for v in row) for row in a]
    Path(path).write_text("\n".join(lines) + "\n")


def read_labeling(path) -> np.ndarray:
    body = [ln for ln in Path(path).read_text().splitlines(keepends=True) if not ln.startswith("#")]
    head = body[0].split() if body else []
    if len(head) < 4 or head[0] != "rows" or head[2] != "cols":
        raise FileFormatError(f"{path}: bad labeling header {body[0] if body else ''!r}")
    rows, cols = int(head[1]), int(head[3])
    vals = np.array(" ".join(body[1:]).split(), dtype=np.int32)
    if vals.size != rows * cols:
        raise FileFormatError(f"{path}: expected {rows * cols} values, got {vals.size}")
    return vals.reshape(rows, cols)
