"""Find the first small case where the default solver disagrees with the oracle or times out."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("GZ_WATCHDOG_MS", "2000")
import numpy as np
import paper_1803_01516_b200 as gz
import paper_1803_01516_b200._lib
from oracle import oracle as o

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 300):
    rows, cols, m = int(rng.integers(1, 8)), int(rng.integers(1, 8)), int(rng.integers(2, 17))
    vol = rng.integers(0, 200, (rows, cols, m)).astype(np.int64)
    pen, inh, hard = int(rng.integers(0, 9)), int(rng.integers(0, 80)), bool(rng.integers(5) == 0)
    win = bool(rng.integers(3) == 0)
    lo = hi = None
    if win:
        lo = rng.integers(0, m, rows * cols).astype(np.int32)
        hi = np.minimum(lo + rng.integers(0, m, rows * cols), m - 1).astype(np.int32)
    p = gz.EnergyParams(pen, inh, hard)
    t0 = time.time()
    try:
        net = gz.build_network(vol, p, lo, hi)
        r = gz.maxflow_push_relabel(net)
        err = None
    except gz._lib.GazecutError as ex:  # noqa
        r, err = None, ex
    onet = o.build_network(vol, pen, p.inhibit_capacity, lo, hi)
    flow, energy, lab, side, st = o.maxflow_push_relabel(onet)
    ok = r is not None and r.flow == flow and np.array_equal(r.labeling, lab)
    if not ok:
        bad += 1
        print(f"case {i}: shape {vol.shape} pen {pen} inh {inh} hard {hard} win {win} err {err} "
              f"got {None if r is None else (r.flow, r.stats['sweeps'], r.stats['pulses'])} want {flow} t {time.time()-t0:.2f}", flush=True)
        if bad == 1:
            np.savez("gpurun_out/bad_case.npz", vol=vol, lo=lo if lo is not None else np.zeros(0), hi=hi if hi is not None else np.zeros(0),
                     params=np.array([pen, inh, int(hard)]))
        if bad >= 5:
            break
print("bad", bad)
