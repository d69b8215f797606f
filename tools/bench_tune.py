"""Bench-level schedule tuning: 64 C1 pairs per call, pairs/s per env combination
(same workload as bench.py's value, device-resident inputs, L2 flushed).
python tools/bench_tune.py 'K=12,BFS_CAP=48,KTAIL=96;K=16,...'"""
import itertools, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import bench
import paper_1803_01516_b200 as gz

P = 64
left, right = bench.scenes(list(range(1000, 1000 + 2 * P)))
L = torch.from_numpy(left).cuda(); R = torch.from_numpy(right).cuda()
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for spec in sys.argv[1].split(";"):
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    for k in list(os.environ):
        if k.startswith("GZ_"):
            del os.environ[k]
    for k, v in env.items():
        os.environ["GZ_" + k] = v
    rates = []
    for rep in range(4):
        s = slice((rep % 2) * P, (rep % 2) * P + P)
        flush.fill_(rep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lab, st = solver.solve(L[s], R[s])
        e1.record(); e1.synchronize()
        if rep > 0:
            rates.append(P / (e0.elapsed_time(e1) / 1e3))
        if rep == 0 and ref is None:
            ref = lab.clone()
        if rep % 2 == 0:
            assert torch.equal(lab, ref), spec
    print(f"{spec:45s} {np.mean(rates):7.1f} pairs/s (min {min(rates):.1f} max {max(rates):.1f})", flush=True)
