"""C5 (3840x2160, 256 labels) exact solve as row bands:
band k on GPU k of the visible devices (or `--bands N --same-gpu` to put N bands
on cuda:0).  Prints flow, energy (certificate: flow == energy of the extracted
labeling) and device time; the one-GPU solve's flow is 170,519,322.

python tools/c5_bands.py [--bands N] [--same-gpu] [--size W H M]"""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1803_01516_b200 as gz

ap = argparse.ArgumentParser()
ap.add_argument("--bands", type=int, default=0)
ap.add_argument("--same-gpu", action="store_true")
ap.add_argument("--size", type=int, nargs=3, default=(3840, 2160, 256))
ap.add_argument("--dmax", type=int, default=511)
a = ap.parse_args()
w, h, m = a.size
n = a.bands or torch.cuda.device_count()
devices = [0] * n if a.same_gpu else list(range(n))
t0 = time.time()
sc = gz.make_scene(0, w, h, 11, a.dmax)
cub = gz.cuboid_from_disparity_range(w, h, 11, a.dmax, num_labels=m)
vol = gz.sad_volume_device(sc.left, sc.right, cub).cpu().numpy()
print("volume", vol.shape, "ready in", round(time.time() - t0, 1), "s; devices", devices, flush=True)
t0 = time.time()
r = gz.solve_exact_bands(vol, gz.EnergyParams(14, 1023), devices=devices)
st = r.stats
print("flow", r.flow, "energy", r.energy, "labeling_energy", st["labeling_energy"], "device_ms", round(st["device_ms"], 1),
      "wall_s", round(time.time() - t0, 1), "sweeps", st["sweeps"], "pulses", st["pulses"], "bfs", st["bfs_passes"],
      "phase_ms", st["phase_ms"], flush=True)
