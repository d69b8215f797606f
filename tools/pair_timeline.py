"""Timeline of batched pair solves (GZ_PAIR_TIMELINE): when the first launch's
queue ran dry, when the tail launch started, when the last pairs finished, and
the host phases of the call next to the CUDA-event time around it -- where a
batch's step time goes.
python tools/pair_timeline.py [reps]   (run under gpurun)"""
import os, sys, time
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
path = os.path.join(ROOT, "gpurun_out", "pair_timeline.txt")
if os.path.exists(path):
    os.remove(path)
os.environ["GZ_PAIR_TIMELINE"] = path
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1803_01516_b200 as gz
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = 1184
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
L = np.empty((n, 288, 384, 3), np.uint8); R = np.empty_like(L)
for i in range(n):
    sc = gz.make_scene(i); L[i], R[i] = sc.left, sc.right
Ld, Rd = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3)
solver.solve(Ld, Rd)
torch.cuda.synchronize()
ev, wall = [], []
if os.environ.get("TL_NOGC"):
    import gc
    gc.collect()
    gc.disable()
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(); lab, st = solver.solve(Ld, Rd); e1.record(); e1.synchronize()
    wall.append((time.perf_counter() - t) * 1e3)
    ev.append(e0.elapsed_time(e1))
blocks, cur = [], None
for line in open(path):
    f = line.split()
    if f[0] == "batch":
        cur = {"hdr": dict(zip(f[0::2], map(int, f[1::2]))), "pairs": []}
        blocks.append(cur)
    else:
        cur["pairs"].append((int(f[1]), int(f[2]), int(f[3])))
for k, blk in enumerate(blocks[1:]):   # (the first block is the warm-up)
    h, ps = blk["hdr"], blk["pairs"]
    b1 = h["batch1"]
    t0 = min(p[1] for p in ps)
    ms = lambda t: (t - t0) * 1e-6
    main = [p for p in ps if p[0] < b1]
    tail = [p for p in ps if p[0] >= b1]
    end = max(p[2] for p in ps)
    print(f"event {ev[k]:7.1f} wall {wall[k]:7.1f} | device: dry {ms(h['dry']):7.1f} tail start {ms(h['tail_start']):7.1f} "
          f"main end {ms(max(p[2] for p in main)):7.1f} tail end {ms(max(p[2] for p in tail)) if tail else 0:7.1f} | "
          f"host: launched {h['h_launch_us'] / 1e3:6.1f} tail launched {h['h_tail_us'] / 1e3:7.1f} copies queued {h['h_copy_us'] / 1e3:7.1f} synced {h['h_sync_us'] / 1e3:7.1f} ms | "
          f"events: k1 end {h['ev_k1_us'] / 1e3:7.1f} k2 end {h['ev_k2_us'] / 1e3:7.1f} stats copied {h['ev_end_us'] / 1e3:7.1f}")
