"""Batched pair solves (gz_solve_pairs) vs the reference's C1 fixtures and the
per-pair solve path: flows, energies and labelings must agree bit for bit."""
import hashlib, json, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1803_01516_b200 as gz
G = json.load(open(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests/golden/golden.json")))
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = np.empty((n, 288, 384, 3), np.uint8); R = np.empty_like(L)
for i in range(n):
    sc = gz.make_scene(i); L[i], R[i] = sc.left, sc.right
solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3)
lab, st = solver.solve(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda())
torch.cuda.synchronize()
t = time.perf_counter(); lab, st = solver.solve(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()); torch.cuda.synchronize()
dt = time.perf_counter() - t
sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
bad = 0
for i, want in enumerate(G["c1_exact"][:min(n, 8)]):
    ok = st[i]["flow"] == want["flow"] and sha(lab[i].cpu().numpy()) == want["labeling"]
    bad += not ok
print(f"{n} pairs in {dt*1e3:.1f} ms -> {n/dt:.1f} pairs/s; fixture mismatches {bad}; mean pair ms {np.mean([s['device_ms'] for s in st]):.1f}",
      "sweeps", np.mean([s['sweeps'] for s in st]), "pulses", np.mean([s['pulses'] for s in st]),
      "bfs", np.mean([s['bfs_passes'] for s in st]), "reach", np.mean([s['reach_passes'] for s in st]),
      {k: round(float(np.mean([s['phase_ms'][k] for s in st])), 2) for k in st[0]['phase_ms']})
