"""Schedule exploration: C1 exact solve under different (bfs_cap, pulses) knobs."""
import sys, time, itertools
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1803_01516_b200 as gz
from paper_1803_01516_b200.maxflow import _run

seeds = [int(s) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0"])]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 16
caps = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["-1", "16", "32", "64", "128", "256"])]
Ks = [int(x) for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["4", "8", "12", "24", "48", "96"])]
for seed in seeds:
    sc = gz.make_scene(seed)
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=m)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    net = gz.build_network(vol, gz.EnergyParams(14, 1023))
    ref = None
    for cap, K in itertools.product(caps, Ks):
        lab, st = _run(net, K, None, True, cap)
        labn = lab.cpu().numpy()
        if ref is None:
            ref = (st.flow, labn)
        ok = st.flow == ref[0] and np.array_equal(labn, ref[1]) and st.labeling_energy == st.flow
        print(f"seed {seed} m {m} cap {cap:4d} K {K:3d}: {st.ms_total:8.2f} ms sweeps {st.sweeps:3d} pulses {st.pulses:4d} "
              f"bfs {st.bfs_passes:5d} reach {st.reach_passes:3d} ok {ok} phases " + " ".join(f"{x:.2f}" for x in st.ms_phase), flush=True)
