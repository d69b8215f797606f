"""Device plumbing: GPU check, uploads, workspaces, stream handles.

PyTorch is used only for device memory and streams; every computation on
the solve path runs in libgazecut_b200.so.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

INT32_MAX = 2**31 - 1


def require_gpu() -> torch.device:
    """The CUDA device to run on; raises if there is no sm_100 GPU (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError("gazecut_b200 needs an sm_100 (B200) GPU; there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device())
    major, _ = torch.cuda.get_device_capability(dev)
    if major != 10:
        raise RuntimeError(f"gazecut_b200 is built for sm_100a; device capability is {major}.x")
    _lib.lib()  # fail loudly if the extension is missing
    return dev


def stream_ptr() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def as_device_i32(a, name: str = "array") -> torch.Tensor:
    """Contiguous int32 CUDA tensor from a numpy array / tensor, range-checked."""
    dev = require_gpu()
    if isinstance(a, torch.Tensor):
        t = a.to(dev)
        if t.dtype != torch.int32:
            if t.numel() and (int(t.min()) < -INT32_MAX or int(t.max()) > INT32_MAX):
                raise ValueError(f"{name} values exceed the int32 device representation")
            t = t.to(torch.int32)
        return t.contiguous()
    arr = np.asarray(a)
    if arr.dtype != np.int32:
        if arr.size and (arr.min() < -INT32_MAX or arr.max() > INT32_MAX):
            raise ValueError(f"{name} values exceed the int32 device representation")
        arr = arr.astype(np.int32)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev, non_blocking=False)


def as_device_u8(a) -> torch.Tensor:
    dev = require_gpu()
    if isinstance(a, torch.Tensor):
        return a.to(dev, dtype=torch.uint8).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.uint8))).to(dev)


_WS: dict = {}
_WS_GEN = [0]


def workspace(nbytes: int) -> torch.Tensor:
    """A cached device workspace of at least ``nbytes`` (per device).  Every
    call starts a new generation: state a solve left in the workspace is valid
    only while the generation it was solved in is current."""
    dev = require_gpu()
    buf = _WS.get(dev.index)
    if buf is None or buf.numel() < nbytes:
        _WS[dev.index] = buf = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
    _WS_GEN[0] += 1
    return buf


def workspace_generation() -> int:
    return _WS_GEN[0]


_CSR_WS: dict = {}


def csr_workspace(nbytes: int) -> torch.Tensor:
    """Workspace of the CSR kernels (separate from the grid solver's)."""
    dev = require_gpu()
    buf = _CSR_WS.get(dev.index)
    if buf is None or buf.numel() < nbytes:
        _CSR_WS[dev.index] = buf = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
    return buf
