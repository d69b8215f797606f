"""Lone-solve A/B of an env knob: mean device ms over seeds x reps on a config.

python tools/lone_ab.py CFG KNOB v1,v2 [seeds] [reps]   e.g. C1 GZ_WORKLIST 0,1 8 3"""
import os, sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_01516_b200 as gz
cfgs = {"C1": (384, 288, 10, 28, 16), "C24": (384, 288, 10, 28, 24), "C2": (450, 375, 11, 59, 60),
        "C3q": (960, 540, 11, 255, 128)}
name, knob, vals = sys.argv[1], sys.argv[2], sys.argv[3].split(",")
nseed = int(sys.argv[4]) if len(sys.argv) > 4 else 4
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
w, h, dmin, dmax, m = cfgs[name]
vols = []
for s in range(nseed):
    sc = gz.make_scene(s, w, h, dmin, dmax)
    vols.append(gz.sad_volume_device(sc.left, sc.right, gz.cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)))
p = gz.EnergyParams(14, 1023)
gz.solve_exact(vols[0], p)  # warm
res = {v: [] for v in vals}
for r in range(reps):
    for v in vals:
        os.environ[knob] = v
        for vol in vols:
            res[v].append(gz.solve_exact(vol, p).stats["device_ms"])
for v in vals:
    xs = res[v]
    print(f"{name} {knob}={v}: mean {statistics.mean(xs):.3f} ms median {statistics.median(xs):.3f} "
          f"min {min(xs):.3f} max {max(xs):.3f} (n={len(xs)})", flush=True)
