"""Time C2 (450x375x60) and C3 (1920x1080x128) exact solves; C2 against the survey golden flow."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1803_01516_b200 as gz
which = sys.argv[1:] or ["C2"]
cfgs = {"C2": (450, 375, 11, 59, 60, 2217255), "C3": (1920, 1080, 11, 255, 128, None)}
for name in which:
    w, h, dmin, dmax, m, golden = cfgs[name]
    t0 = time.time()
    sc = gz.make_scene(0, w, h, dmin, dmax)
    cub = gz.cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
    print(name, "scene", round(time.time() - t0, 1), "s; sites", cub.site_shape, flush=True)
    vol = gz.sad_volume_device(sc.left, sc.right, cub)
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.time()
        r = gz.solve_exact(vol, gz.EnergyParams(14, 1023))
        torch.cuda.synchronize()
        st = r.stats
        print(name, "rep", rep, "flow", r.flow, "energy", r.energy, "golden", golden, "ok", golden is None or r.flow == golden,
              "device_ms", round(st["device_ms"], 2), "wall", round(time.time() - t0, 2), "sweeps", st["sweeps"], "pulses",
              st["pulses"], "bfs", st["bfs_passes"], "phase", st["phase_ms"], flush=True)
