"""Phase breakdown of the hierarchy modes on the 24-label scene."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_01516_b200 as gz
from paper_1803_01516_b200 import hierarchy as H
sc = gz.make_scene(0)
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
for rep in range(2):
    for name, fn in (("l1b3", lambda: gz.solve_level1(vol, p, 3)), ("l2b3", lambda: gz.solve_level2(vol, p, 3))):
        r = fn()
        s = r.stats
        print(name, "coarse_ms", round(s["coarse_device_ms"], 3), "fine_ms", round(s["device_ms"], 3), "sweeps", s["sweeps"],
              "pulses", s["pulses"], "bfs", s["bfs_passes"], "phase", s["phase_ms"], "window", round(s["mean_window"], 2), flush=True)
cv = H.coarsen_device(gz.sad_volume_device(sc.left, sc.right, cub).contiguous(), 3)
rc = gz.solve_exact(cv, gz.EnergyParams(42, 1023))
print("coarse exact alone", rc.stats["device_ms"], rc.stats["sweeps"], rc.stats["pulses"], rc.stats["phase_ms"])
