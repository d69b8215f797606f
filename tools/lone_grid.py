import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1803_01516_b200 as gz
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
sc = gz.make_scene(0)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
for g in sys.argv[1:]:
    os.environ["GZ_LONE_GRID"] = g
    ts = []
    for _ in range(2):
        r = gz.solve_exact(vol, p)
        ts.append(r.stats["device_ms"])
    print("grid", g, "occ", os.environ.get("GZ_OCC"), "flow", r.flow, "ms", [round(t, 2) for t in ts], "sweeps", r.stats["sweeps"], "pulses", r.stats["pulses"], "bfs", r.stats["bfs_passes"], r.stats["phase_ms"], flush=True)
