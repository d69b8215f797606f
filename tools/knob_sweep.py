"""Schedule-knob sweep for batched pair solves (gz_solve_pairs), one process:
the knobs are environment variables read per call (gz_solver.cu setup_prob).

python tools/knob_sweep.py PAIRS 'NAME=V,NAME2=V2' 'NAME=V' ..."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))

import numpy as np, torch
import paper_1803_01516_b200 as gz
n = int(sys.argv[1])
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
L = np.empty((n, 288, 384, 3), np.uint8); R = np.empty_like(L)
for i in range(n):
    sc = gz.make_scene(1000 + i); L[i], R[i] = sc.left, sc.right
Ld, Rd = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
solver = gz.PairSolver(cub, gz.EnergyParams(14, 1023), 288, 384, 3)
base = {k: v for k, v in os.environ.items() if k.startswith("GZ_")}
solver.solve(Ld, Rd); torch.cuda.synchronize()
ref_flows = None
for cfg in sys.argv[2:] or [""]:
    for k in list(os.environ):
        if k.startswith("GZ_") and k not in base:
            del os.environ[k]
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    ts = []
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        lab, st = solver.solve(Ld, Rd); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    flows = [s["flow"] for s in st]
    if ref_flows is None:
        ref_flows = flows
    ok = flows == ref_flows
    ph = {k: round(float(np.mean([s["phase_ms"][k] for s in st])), 1) for k in ("global_relabel", "pulses")}
    print(f"{cfg or 'default':40s} {n / min(ts):7.1f} pairs/s  pair {np.mean([s['device_ms'] for s in st]):6.1f} ms "
          f"sweeps {np.mean([s['sweeps'] for s in st]):5.2f} pulses {np.mean([s['pulses'] for s in st]):6.1f} {ph} flows_ok={ok}",
          flush=True)
