"""Matching energy: data term on device, pairwise profile, labeling energy.

Mirrors ``gazecut.energy`` (energy.py:1-155).  ``sad_volume`` and
``total_energy`` run as sm_100a kernels (gz_sad_volume / gz_total_energy);
the scalar helpers are host-side definitions of the model.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .geometry import CuboidSpec

UNCUTTABLE = 1 << 56  # energy.py:34


@dataclass(frozen=True)
class EnergyParams:
    """energy.py:37-50."""

    penalty: int = 14
    inhibit: int = 1023
    hard_inhibit: bool = False

    def __post_init__(self):
        if self.penalty < 0 or self.inhibit < 0:
            raise ValueError("penalty and inhibit must be non-negative")

    @property
    def inhibit_capacity(self) -> int:
        return UNCUTTABLE if self.hard_inhibit else self.inhibit

    def _c(self) -> _lib.Energy:
        if self.penalty > 2**30 or self.inhibit > 2**30:
            raise ValueError("penalty/inhibit exceed the int32 device representation")
        return _lib.Energy(int(self.penalty), int(self.inhibit), 1 if self.hard_inhibit else 0)


def data_term(colour_a, colour_b) -> int:
    return int(np.abs(np.asarray(colour_a, np.int64) - np.asarray(colour_b, np.int64)).sum())


def pairwise_term(i: int, j: int, params: EnergyParams) -> int:
    """penalty*|d| + inhibit*(|d|-1) for |d| > 1 (energy.py:60-67)."""
    delta = abs(i - j)
    if delta == 0:
        return 0
    if delta > 1 and params.hard_inhibit:
        return UNCUTTABLE
    return params.penalty * delta + params.inhibit * (delta - 1)


def is_convex_profile(h, max_delta: int) -> bool:
    return all(h(d - 1) - 2 * h(d) + h(d + 1) >= 0 for d in range(-max_delta + 1, max_delta))


def neighbour_pairs(site_shape: tuple[int, int]):
    rows, cols = site_shape
    idx = np.arange(rows * cols).reshape(rows, cols)
    return (np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()]),
            np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()]))


def cuboid_struct(cuboid: CuboidSpec, width: int) -> _lib.Cuboid:
    return _lib.Cuboid(int(width), 0, cuboid.g_min, cuboid.g_extent, cuboid.y_min, cuboid.y_extent,
                       cuboid.d_min, cuboid.num_labels)


def _images(left, right):
    if tuple(left.shape) != tuple(right.shape):
        raise ValueError(f"image shapes differ: {tuple(left.shape)} vs {tuple(right.shape)}")
    if len(left.shape) not in (2, 3):
        raise ValueError("images must be (h, w) or (h, w, channels)")
    h, w = int(left.shape[0]), int(left.shape[1])
    ch = 1 if len(left.shape) == 2 else int(left.shape[2])
    return h, w, ch


def sad_volume_device(left, right, cuboid: CuboidSpec, width: int | None = None) -> torch.Tensor:
    """Data term on device: int32 CUDA tensor (y_extent, g_extent, m)."""
    h, w, ch = _images(left, right)
    width = w if width is None else width
    cuboid.check_consistent(width, h)
    if width > w:
        # the reference gathers columns clipped to [0, width-1] from the images and
        # fails with IndexError past their edge (geometry.py:325-335)
        raise IndexError(f"cuboid width {width} exceeds the image width {w}")
    dl, dr = _dev.as_device_u8(left), _dev.as_device_u8(right)
    out = torch.empty((cuboid.y_extent, cuboid.g_extent, cuboid.num_labels), dtype=torch.int32, device=dl.device)
    cs = cuboid_struct(cuboid, width)
    cs.height = h
    _lib.check(_lib.lib().gz_sad_volume(_dev.ptr(dl), _dev.ptr(dr), h, w, ch, C.byref(cs), _dev.ptr(out),
                                        _dev.stream_ptr()), "gz_sad_volume")
    return out


def sad_volume(left, right, cuboid: CuboidSpec, width: int | None = None) -> np.ndarray:
    """energy.py:83-114: int64 (y_extent, g_extent, num_labels), computed on the GPU."""
    return sad_volume_device(left, right, cuboid, width).cpu().numpy().astype(np.int64)


def total_energy_device(labeling: torch.Tensor, volume: torch.Tensor, params: EnergyParams) -> int:
    rows, cols, m = (int(s) for s in volume.shape)
    out = torch.zeros(2, dtype=torch.int64, device=volume.device)
    en = params._c()
    _lib.check(_lib.lib().gz_total_energy(_dev.ptr(labeling), _dev.ptr(volume), rows, cols, m, C.byref(en),
                                          _dev.ptr(out), _dev.stream_ptr()), "gz_total_energy")
    e, viol = (int(x) for x in out.cpu())
    return UNCUTTABLE if viol else e


def total_energy(labeling, volume, params: EnergyParams) -> int:
    """energy.py:129-155, evaluated on the GPU."""
    lab = np.asarray(labeling) if not isinstance(labeling, torch.Tensor) else labeling
    rows, cols, m = (int(s) for s in volume.shape)
    if tuple(lab.shape) != (rows, cols):
        raise ValueError(f"labeling shape {tuple(lab.shape)} != site grid {(rows, cols)}")
    lmin, lmax = int(lab.min()), int(lab.max())
    if lmin < 0 or lmax >= m:
        raise ValueError("label outside volume range")
    return total_energy_device(_dev.as_device_i32(lab, "labeling"), _dev.as_device_i32(volume, "volume"), params)
