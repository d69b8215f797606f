"""Lone C1 solves (one pair on all SMs), mean device ms over seeds 0-7, per
environment configuration (knobs are read per solve).

python tools/lone_seeds.py 'NAME=V,NAME2=V2' ..."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1803_01516_b200 as gz
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
vols = []
for sd in range(8):
    sc = gz.make_scene(sd)
    vols.append(gz.sad_volume_device(sc.left, sc.right, cub))
p = gz.EnergyParams(14, 1023)
base = {k for k in os.environ if k.startswith("GZ_")}
for cfg in sys.argv[1:] or [""]:
    for k in list(os.environ):
        if k.startswith("GZ_") and k not in base:
            del os.environ[k]
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    ms, ph = [], []
    for v in vols:
        gz.solve_exact(v, p)
        r = gz.solve_exact(v, p)
        ms.append(r.stats["device_ms"])
        ph.append(r.stats["phase_ms"])
    agg = {k: round(float(np.mean([x[k] for x in ph])), 3) for k in ("global_relabel", "pulses", "mask_build")}
    print(f"{cfg or 'default':36s} mean {np.mean(ms):6.3f} ms  min {min(ms):6.3f} max {max(ms):6.3f} {agg}", flush=True)
