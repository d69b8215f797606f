"""Device-timed batched pair solves: 1184 C1 pairs (the bench's block) with
device-resident images, CUDA events around each solve, 1 warm-up + N timed.
Prints the per-solve ms, pairs/s and the mean per-pair device ms (CTR_NS).
python tools/pairs_time.py [n_pairs] [reps]"""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1803_01516_b200 as gz
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
L = np.empty((n, 288, 384, 3), np.uint8); R = np.empty_like(L)
for i in range(n):
    sc = gz.make_scene(i); L[i], R[i] = sc.left, sc.right
Ld, Rd = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3)
solver.solve(Ld, Rd)
torch.cuda.synchronize()
ms, pm, mx = [], [], []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); lab, st = solver.solve(Ld, Rd); e1.record(); e1.synchronize()
    ms.append(e0.elapsed_time(e1)); pm.append(np.mean([s["device_ms"] for s in st])); mx.append(max(s["device_ms"] for s in st))
tag = os.environ.get("TAG", "")
print(f"{tag:24s} solve ms {' '.join(f'{x:.1f}' for x in ms)} -> {n / (np.mean(ms) / 1e3):.1f} pairs/s; mean pair ms {np.mean(pm):.1f}; max pair ms {' '.join(f'{x:.0f}' for x in mx)}")
