"""Shared helper for the schedule tools: one device solve with explicit knobs."""
import ctypes as C, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1803_01516_b200 import _lib, _dev


def run(net, K, cap, flags=0):
    rows, cols = net.site_shape
    L = _lib.lib()
    nb = L.gz_workspace_bytes(rows, cols, net.num_labels)
    ws = _dev.workspace(nb)
    lab = torch.empty(rows * cols, dtype=torch.int32, device="cuda")
    st = _lib.Stats()
    en = net.params._c()
    sc = _lib.Sched(K, 0, cap, flags)
    rc = L.gz_solve_volume(_dev.ptr(net.volume), rows, cols, net.num_labels, C.byref(en), C.byref(sc), None, None,
                           _dev.ptr(lab), C.byref(st), _dev.ptr(ws), nb, _dev.stream_ptr())
    _lib.check(rc, "solve")
    return lab.cpu().numpy(), st
