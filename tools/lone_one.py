"""One lone C1 solve (seed 0) after a warm-up, for ncu captures of the lone
tilesolve launch: python tools/lone_one.py [seed]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_01516_b200 as gz
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
sc = gz.make_scene(seed)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
for _ in range(2):
    r = gz.solve_exact(vol, gz.EnergyParams(14, 1023))
print("flow", r.flow, "device_ms", r.stats["device_ms"], r.stats["phase_ms"])
