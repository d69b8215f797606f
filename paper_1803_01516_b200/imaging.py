"""Ground truth on the device (imaging.py:133-201 of the reference).

Only the accuracy path is here: ``GroundTruthDepth`` and
``ground_truth_to_depth`` (gz_ground_truth_to_depth).  Image file I/O
(netpbm, disparity PNGs) stays host-side tooling, out of scope."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _dev, _lib
from .geometry import CuboidSpec


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
