"""C5 (3840x2160, 256 labels) exact solve on ONE B200: data term, solve, and the
optimality certificate (flow == energy of the extracted labeling)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import hashlib, numpy as np, torch
import paper_1803_01516_b200 as gz
t0 = time.time()
sc = gz.make_scene(0, 3840, 2160, 11, 511)
cub = gz.cuboid_from_disparity_range(3840, 2160, 11, 511, num_labels=256)
print("scene", round(time.time() - t0, 1), "s; sites", cub.site_shape, flush=True)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
torch.cuda.synchronize()
print("volume", tuple(vol.shape), "sha", hashlib.sha256(vol.cpu().numpy().astype(np.int64).tobytes()).hexdigest(), flush=True)
t0 = time.time()
r = gz.solve_exact(vol, gz.EnergyParams(14, 1023))
torch.cuda.synchronize()
st = r.stats
print("C5 flow", r.flow, "energy", r.energy, "labeling_energy", st["labeling_energy"], "device_ms", st["device_ms"],
      "wall", round(time.time() - t0, 1), "sweeps", st["sweeps"], "pulses", st["pulses"], "bfs", st["bfs_passes"],
      "phase", st["phase_ms"], flush=True)
