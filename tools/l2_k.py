"""Level-2 energy / time vs capped pulses per sweep (GZ_CAPPED_K) on the 24-label
scene; reference l2b3 energy 790883, level-1 790627.  python tools/l2_k.py 12,24,36,48"""
import os, sys, statistics
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1803_01516_b200 as gz
sc = gz.make_scene(0)
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
for b in (2, 3):
    for K in sys.argv[1].split(","):
        os.environ["GZ_CAPPED_K"] = K
        ts, es = [], set()
        for _ in range(4):
            r = gz.solve_level2(vol, p, b)
            ts.append(r.stats["device_ms_total"])
            es.add(r.energy)
        print(f"b {b} K {K:>3}: energy {sorted(es)} median device_total {statistics.median(ts):.2f} ms "
              f"(fine pulses {r.stats['pulses']}, sweeps {r.stats['sweeps']}, converged {r.stats['converged']})", flush=True)
