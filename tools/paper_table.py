"""The paper's Table 1 modes on the reference's 24-label
Tsukuba-shaped synthetic scene (seed 0, 384x288, dis 10..28): exact, level-1
b=2 / b=3, level-2 b=3.  Prints energy and device time (solver kernels,
CUDA events) and wall time per mode, median of 5 runs after 2 warm-ups."""
import statistics, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1803_01516_b200 as gz

sc = gz.make_scene(0)
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
modes = {"exact": lambda: gz.solve_exact(vol, p), "l1b2": lambda: gz.solve_level1(vol, p, 2),
         "l1b3": lambda: gz.solve_level1(vol, p, 3), "l2b3": lambda: gz.solve_level2(vol, p, 3)}
paper = {"exact": 122, "l1b2": 14, "l1b3": 14, "l2b3": 5}
for name, fn in modes.items():
    for _ in range(2):
        fn()
    dev, wall, en = [], [], None
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(r.stats.get("device_ms_total", r.stats["device_ms"]))
        en = r.energy
    print(f"{name}: energy {en} device {statistics.median(dev):.3f} ms wall {statistics.median(wall):.3f} ms "
          f"(paper GTX1080 {paper[name]} ms)", flush=True)
