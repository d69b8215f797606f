"""Level-2 (capped) quality vs pulses per sweep on the 24-label scene (reference l2b3 = 790883)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1803_01516_b200 as gz
sc = gz.make_scene(0)
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
for K in [int(x) for x in sys.argv[1].split(",")]:
    for ms in (8,):
        r = gz.solve_level2(vol, p, 3, rounds_per_sweep=K, max_sweeps=ms)
        r = gz.solve_level2(vol, p, 3, rounds_per_sweep=K, max_sweeps=ms)
        print(f"K {K:4d} max_sweeps {ms}: energy {r.energy} converged {r.stats['converged']} device_total "
              f"{r.stats['device_ms_total']:.2f} ms (fine {r.stats['device_ms']:.2f}) pulses {r.stats['pulses']}", flush=True)
