"""Run the golden random cases through the v1 (forced with GZ_SCHED_V1) and the default v4 solver; print the first mismatches."""
import ctypes as C, json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np, torch
import paper_1803_01516_b200 as gz
from paper_1803_01516_b200 import _lib, _dev

def run(net, flags):
    rows, cols = net.site_shape
    L = _lib.lib()
    nb = L.gz_workspace_bytes(rows, cols, net.num_labels)
    ws = _dev.workspace(nb)
    lab = torch.empty(rows * cols, dtype=torch.int32, device="cuda")
    st = _lib.Stats()
    en = net.params._c()
    sc = _lib.Sched(12, 0, 0, flags)
    lo = _dev.ptr(net.lo) if net.lo is not None else None
    hi = _dev.ptr(net.hi) if net.hi is not None else None
    rc = L.gz_solve_volume(_dev.ptr(net.volume), rows, cols, net.num_labels, C.byref(en), C.byref(sc), lo, hi,
                           _dev.ptr(lab), C.byref(st), _dev.ptr(ws), nb, _dev.stream_ptr())
    return rc, lab.cpu().numpy(), st

G = json.loads((ROOT / "tests/golden/golden.json").read_text())
arr = np.load(ROOT / "tests/golden/random_cases.npz")
bad = 0
for i, meta in enumerate(G["random_cases"]):
    p = gz.EnergyParams(meta["penalty"], meta["inhibit"], meta["hard"])
    lo = arr[f"lo{i}"] if meta["windowed"] else None
    hi = arr[f"hi{i}"] if meta["windowed"] else None
    net = gz.build_network(arr[f"vol{i}"], p, lo, hi)
    out = []
    for fl in (_lib.GZ_SCHED_V1, 0):
        rc, lab, st = run(net, fl)
        out.append((rc, st.flow, st.sweeps, st.pulses, st.bfs_passes, st.pushes, st.relabels, st.presaturated, st.reach_passes))
    if out[0][1] != out[1][1] or out[1][1] != meta["flow"]:
        bad += 1
        print(i, arr[f"vol{i}"].shape, meta["windowed"], meta["hard"], "want", meta["flow"], "v1", out[0], "v4", out[1], flush=True)
        if bad > 8:
            break
print("bad", bad)
