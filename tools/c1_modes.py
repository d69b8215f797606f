"""C1 (384x288x16, seed 0) exact / level-1 / level-2 device times (median of 5 after 2 warm-ups)."""
import statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_01516_b200 as gz
sc = gz.make_scene(0)
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
for name, fn in (("exact", lambda: gz.solve_exact(vol, p)), ("l1b2", lambda: gz.solve_level1(vol, p, 2)),
                 ("l1b4", lambda: gz.solve_level1(vol, p, 4)), ("l2b2", lambda: gz.solve_level2(vol, p, 2))):
    for _ in range(2):
        fn()
    dev, en = [], None
    for _ in range(5):
        r = fn()
        dev.append(r.stats.get("device_ms_total", r.stats["device_ms"]))
        en = r.energy
    print(f"C1 {name}: energy {en} device {statistics.median(dev):.3f} ms", flush=True)
