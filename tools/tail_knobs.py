"""Mean C1 solve time over seeds for schedule knobs: python tools/tail_knobs.py 'K,cap,ktail,after;...'"""
import os, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1803_01516_b200 as gz
seeds = list(range(8))
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
sc = [gz.make_scene(s) for s in seeds]
L = torch.from_numpy(np.stack([s.left for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.right for s in sc])).cuda()
os.environ["GZ_PAIR_CONC"] = "1"
ref = None
for spec in sys.argv[1].split(";"):
    K, cap, kt, ta = spec.split(",")
    solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3, rounds_per_sweep=int(K), bfs_cap=int(cap))
    os.environ["GZ_KTAIL"], os.environ["GZ_TAIL_AFTER"] = kt, ta
    ms, sw, pl, lv = [], [], [], []
    for rep in range(3):
        lab, st = solver.solve(L, R)
        if ref is None:
            ref = lab.clone()
        assert torch.equal(lab, ref)
        ms += [s["device_ms"] for s in st]; sw += [s["sweeps"] for s in st]; pl += [s["pulses"] for s in st]
        lv += [s["bfs_passes"] for s in st]
    ph = {k: round(statistics.mean(s["phase_ms"][k] for s in st), 3) for k in st[0]["phase_ms"]}
    print(f"K {K:>3} cap {cap:>3} ktail {kt:>3} after {ta}: {statistics.mean(ms):.3f} ms (min {min(ms):.3f} max {max(ms):.3f}) sweeps {statistics.mean(sw):.1f} "
          f"pulses {statistics.mean(pl):.1f} levels {statistics.mean(lv):.0f} {ph}", flush=True)
