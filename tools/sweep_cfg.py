"""Schedule exploration on a BASELINE config: python tools/sweep_cfg.py C2 H1,H2 cap1,cap2 K1,K2"""
import itertools, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1803_01516_b200 as gz
from _solve import run
cfgs = {"C1": (384, 288, 10, 28, 16), "C2": (450, 375, 11, 59, 60), "C3": (1920, 1080, 11, 255, 128),
        "C24": (384, 288, 10, 28, 24), "C3q": (960, 540, 11, 255, 128), "C3e": (480, 270, 11, 255, 128),
        "C1m128": (384, 288, 10, 28, 128), "C3m32": (1920, 1080, 11, 255, 32)}
name = sys.argv[1]
w, h, dmin, dmax, m = cfgs[name]
Hs = [int(x) for x in sys.argv[2].split(",")]
caps = [int(x) for x in sys.argv[3].split(",")]
Ks = [int(x) for x in sys.argv[4].split(",")]
sc = gz.make_scene(0, w, h, dmin, dmax)
cub = gz.cuboid_from_disparity_range(w, h, dmin, dmax, num_labels=m)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
net = gz.build_network(vol, gz.EnergyParams(14, 1023))
ref = None
for H, cap, K in itertools.product(Hs, caps, Ks):
    if H > 0:
        os.environ["GZ_BFS_H"] = str(H)
    else:   # 0: the library's residency-based default
        os.environ.pop("GZ_BFS_H", None)
    try:
        lab, st = run(net, K, cap)
    except Exception as ex:  # noqa
        print(f"{name} H {H} cap {cap} K {K}: {ex}", flush=True)
        continue
    if ref is None:
        ref = (st.flow, lab)
    ok = st.flow == ref[0] and np.array_equal(lab, ref[1]) and st.labeling_energy == st.flow
    print(f"{name} H {H:2d} cap {cap:5d} K {K:3d}: {st.ms_total:9.2f} ms flow {st.flow} sweeps {st.sweeps:5d} pulses {st.pulses:6d} "
          f"bfs {st.bfs_passes:7d} ok {ok} phases " + " ".join(f"{x:.2f}" for x in st.ms_phase), flush=True)
