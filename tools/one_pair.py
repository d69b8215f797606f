"""Solve C1 pairs through PairSolver (for ncu captures): python tools/one_pair.py [n_solves] [pairs_per_call]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1803_01516_b200 as gz
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
per = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
sc = [gz.make_scene(s) for s in range(per)]
L = torch.from_numpy(np.stack([s.left for s in sc])).cuda()
R = torch.from_numpy(np.stack([s.right for s in sc])).cuda()
solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3)
for i in range(n):
    lab, st = solver.solve(L, R)
    print(i, [(s["flow"], round(s["device_ms"], 3), s["phase_ms"]) for s in st], flush=True)
