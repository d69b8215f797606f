"""v4 schedule exploration: C1 exact solve over (BFS halo H, bfs_cap, pulses per sweep)."""
import ctypes as C, itertools, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1803_01516_b200 as gz
from paper_1803_01516_b200 import _lib, _dev

from _solve import run

seeds = [int(s) for s in sys.argv[1].split(",")]
Hs = [int(x) for x in sys.argv[2].split(",")]
caps = [int(x) for x in sys.argv[3].split(",")]
Ks = [int(x) for x in sys.argv[4].split(",")]
m = int(sys.argv[5]) if len(sys.argv) > 5 else 16
for seed in seeds:
    sc = gz.make_scene(seed)
    cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=m)
    vol = gz.sad_volume(sc.left, sc.right, cub)
    net = gz.build_network(vol, gz.EnergyParams(14, 1023))
    ref_lab, ref = run(net, 12, 0, _lib.GZ_SCHED_V2)
    print(f"seed {seed} v2 ref: {ref.ms_total:.2f} ms flow {ref.flow}", flush=True)
    for H, cap, K in itertools.product(Hs, caps, Ks):
        os.environ["GZ_BFS_H"] = str(H)
        best = None
        for rep in range(2):
            lab, st = run(net, K, cap)
            best = st.ms_total if best is None else min(best, st.ms_total)
        ok = st.flow == ref.flow and np.array_equal(lab, ref_lab) and st.labeling_energy == st.flow
        print(f"seed {seed} H {H:2d} cap {cap:4d} K {K:3d}: {best:7.2f} ms sweeps {st.sweeps:3d} pulses {st.pulses:4d} "
              f"bfs {st.bfs_passes:5d} reach {st.reach_passes:3d} ok {ok} phases " + " ".join(f"{x:.2f}" for x in st.ms_phase), flush=True)
