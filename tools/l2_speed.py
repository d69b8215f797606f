"""Level-2 speed / quality trade on the 24-label ladder scene (PAPER.md:437-457,
reference recorded energies pkg/test_output.txt:24: L1b2 785090, L1b3 790627,
L2b3 790883): device ms and energy per capped pulses-per-sweep K (GZ_CAPPED_K)
and sweep cap.

python tools/l2_speed.py K1 K2 ..."""
import os, statistics, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1803_01516_b200 as gz
sc = gz.make_scene(0)
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=24)
vol = gz.sad_volume_device(sc.left, sc.right, cub)
p = gz.EnergyParams(14, 1023)
for b in (2, 3):
    r = gz.solve_level1(vol, p, b)
    dev = statistics.median(gz.solve_level1(vol, p, b).stats["device_ms_total"] for _ in range(3))
    print(f"L1 b{b}: energy {r.energy} device {dev:.3f} ms", flush=True)
for k in sys.argv[1:]:
    os.environ["GZ_CAPPED_K"] = k
    for b in (2, 3):
        for ms in (8, 4, 2):
            rs = [gz.solve_level2(vol, p, b, max_sweeps=ms) for _ in range(4)]
            dev = statistics.median(r.stats["device_ms_total"] for r in rs[1:])
            print(f"K={k} b{b} max_sweeps={ms}: energy {rs[-1].energy} device {dev:.3f} ms "
                  f"(fine {statistics.median(r.stats['device_ms'] for r in rs[1:]):.3f}) sweeps {rs[-1].stats['sweeps']} "
                  f"pulses {rs[-1].stats['pulses']} converged {rs[-1].stats['converged']}", flush=True)
