#!/usr/bin/env python
"""Benchmark: exact stereo graph cut of Tsukuba-shaped pairs on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--pairs P] [--impl ours|reference]

Metric (BASELINE.json): ms per stereo pair (Tsukuba 384x288x16) and pairs/s at
1/2/4/8 B200 vs the CPU reference.  Workload = BASELINE config 4 shape: batches
of Tsukuba-shaped pairs (make_scene(seed), 384x288, dis 10..28, 16 labels,
penalty 14 / inhibit 1023) sharded by pair over ranks, no collectives on the
data path (weak scaling: P pairs per rank per step).  A step = sad_volume +
solve_exact (exact min cut, labels + flow + energy, identity check on device)
for every pair of the rank's batch.  Under torchrun each rank drives one GPU;
the reported time is the max over ranks.  Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"]
W_IMG, H_IMG, DIS_MIN, DIS_MAX, LABELS = 384, 288, 10, 28, 16
PENALTY, INHIBIT = 14, 1023


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def state_bytes(rows: int, cols: int, m: int) -> int:
    """minimal state S = 8 N_int + 4 sites m + 2 nb (m-1) + 2 nb 2 (m-2)."""
    sites = rows * cols
    n_int = sites * (m - 1)
    nb = rows * (cols - 1) + (rows - 1) * cols
    return 8 * n_int + 4 * sites * m + 2 * nb * (m - 1) + 2 * nb * 2 * (m - 2)


def update_bytes(st: dict, rows: int, cols: int, m: int) -> int:
    """SURVEY.md 8(d) algorithmic bytes of one solve: every graph-node update
    (one interior node processed by one push/relabel pulse; counted on the
    device, stats['node_updates']) moves 2S / N_int bytes, S the minimal state
    (47.4 B at C1).  This is the figure roofline.achieved uses."""
    S = state_bytes(rows, cols, m)
    n_int = rows * cols * (m - 1)
    return int(st["node_updates"] * 2 * S / n_int)


def other_bytes(st: dict, rows: int, cols: int, m: int) -> int:
    """Work outside the push/relabel pulses, reported beside (not inside) the
    roofline: a mask build reads the state once and
    writes 13 arc-mask words + 1 excess word per site; a bit-parallel BFS level
    reads 13 mask words + frontier + visited and writes frontier + visited
    (68 B/site; temporally blocked, so most of it stays in shared memory); a
    reach pass moves 76 B/site."""
    S = state_bytes(rows, cols, m)
    sites = rows * cols
    builds = st["sweeps"] + 1
    return int(builds * (S + 56 * sites) + st["bfs_passes"] * 68 * sites + st["reach_passes"] * 76 * sites)


def rank_seeds(rank: int, pairs_per_step: int, steps: int) -> list[int]:
    """C4 sharding: rank r solves its own contiguous block of
    scene seeds, pairs_per_step per step plus one warm-up batch; no pair is
    solved by two ranks and nothing crosses GPUs."""
    return [rank * 100_000 + i for i in range(pairs_per_step * (steps + 1))]


def max_over_ranks(value_ms: float, world: int, device=None) -> float:
    """The job's time is the slowest rank's device time (an all-reduce MAX of one
    float; the only collective in the benchmark, outside the timed region)."""
    if world <= 1:
        return float(value_ms)
    import torch
    import torch.distributed as dist
    t = torch.tensor([value_ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def scenes(seeds):
    from paper_1803_01516_b200 import make_scene
    left = np.empty((len(seeds), H_IMG, W_IMG, 3), np.uint8)
    right = np.empty_like(left)
    for i, s in enumerate(seeds):
        sc = make_scene(int(s), W_IMG, H_IMG, DIS_MIN, DIS_MAX)
        left[i], right[i] = sc.left, sc.right
    return left, right


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_baseline_sample(n_threads: int, seeds):
    """The oracle port of the reference path (sad_volume + solve_exact, CSR build,
    FIFO push-relabel, BFS cut, identity check) on n_threads host threads, one
    pair per thread (ctypes releases the GIL)."""
    from oracle import oracle as o
    from paper_1803_01516_b200 import cuboid_from_disparity_range
    o.build_lib()
    cub = cuboid_from_disparity_range(W_IMG, H_IMG, DIS_MIN, DIS_MAX, num_labels=LABELS)
    left, right = scenes(seeds[:n_threads])
    out = [None] * n_threads

    def work(i):
        vol = o.sad_volume(left[i], right[i], cub.g_min, cub.g_extent, cub.y_min, cub.y_extent, cub.d_min, LABELS)
        out[i] = o.solve_exact(vol, PENALTY, INHIBIT)["flow"]

    threads = [threading.Thread(target=work, args=(i,)) for i in range(n_threads)]
    t0 = time.perf_counter()
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    wall = time.perf_counter() - t0
    return n_threads / wall, wall, out


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    n = min(host_threads(), 32)
    log(f"[reference] oracle port of the reference path on {n} host threads")
    from oracle import oracle as o
    o.build_lib()
    tiny = np.arange(2 * 3 * 4, dtype=np.int64).reshape(2, 3, 4)
    for _ in range(args.warmup):   # native code: warm-up = loading + page-in, kept tiny
        o.solve_exact(tiny, 1, 5)
    # one pair on one core, stage by stage (the 1-core latency split)
    from paper_1803_01516_b200 import cuboid_from_disparity_range
    cub = cuboid_from_disparity_range(W_IMG, H_IMG, DIS_MIN, DIS_MAX, num_labels=LABELS)
    (l1,), (r1,) = scenes([100])
    t0 = time.perf_counter()
    vol = o.sad_volume(l1, r1, cub.g_min, cub.g_extent, cub.y_min, cub.y_extent, cub.d_min, LABELS)
    t1 = time.perf_counter()
    o.solve_exact(vol, PENALTY, INHIBIT)
    t2 = time.perf_counter()
    lat = {"sad_volume": t1 - t0, "solve_exact": t2 - t1, "total": t2 - t0,
           "ms_per_pair": 1000 * (t2 - t0), "seed": 100, "threads": 1}
    log(f"[reference] 1-core latency: {lat}")
    rates, walls = [], []
    for k in range(args.steps):
        rate, wall, flows = cpu_baseline_sample(n, list(range(100 + k * n, 100 + (k + 1) * n)))
        rates.append(rate)
        walls.append(wall)
        log(f"[reference] step {k}: {n} pairs in {wall:.1f} s")
    value = n * len(walls) / sum(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(walls) / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (make_scene seeds, regenerated bit-identically to the reference)",
        "config": {"workload": "C4-shaped batch: Tsukuba 384x288x16 pairs, exact solve", "pairs_per_step": n,
                   "labels": LABELS, "penalty": PENALTY, "inhibit": INHIBIT},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": n, "kind": "port",
                         "sample": f"{n} pairs per step, one per host thread (oracle/gz_oracle.c, C port of "
                                   "sad_volume + solve_exact)"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "latency_1core_s": lat,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--pairs", type=int, default=1184,
                    help="pairs per rank per step (1184 = 8 per team of the batched launch; BASELINE config 4 "
                         "is a 512-pair batch)")
    ap.add_argument("--no-lone", action="store_true", help="skip the lone-pair latency measurement")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=32)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1803_01516_b200 as gz
    from paper_1803_01516_b200 import _lib

    dev = torch.device("cuda", local)
    cub = gz.cuboid_from_disparity_range(W_IMG, H_IMG, DIS_MIN, DIS_MAX, num_labels=LABELS)
    params = gz.EnergyParams(PENALTY, INHIBIT)
    solver = gz.PairSolver(cub, params, H_IMG, W_IMG, 3)
    P = args.pairs
    seeds = rank_seeds(rank, P, args.steps)
    left_h, right_h = scenes(seeds)
    left_d = torch.from_numpy(left_h).to(dev)
    right_d = torch.from_numpy(right_h).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def batch(k):
        j = (k % (args.steps + 1)) * P
        return slice(j, j + P)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up ----
    for w in range(args.warmup):
        s = batch(w)
        solver.solve(left_d[s], right_d[s])
    torch.cuda.synchronize()

    # ---- timed: device-resident inputs ----
    stream = torch.cuda.current_stream()
    step_ms, all_stats = [], []
    barrier()
    with ClockSampler(local) as clocks:
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)          # L2 flush between timed steps (untimed)
            s = batch(k)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            labels, stats = solver.solve(left_d[s], right_d[s])
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            all_stats.extend(stats)
        barrier()
        wall_s = time.perf_counter() - t_wall
    dev_ms = sum(step_ms)
    max_ms = max_over_ranks(dev_ms, world, dev)
    total_pairs = P * args.steps * world
    value = total_pairs / (max_ms / 1000.0)

    # ---- end to end: host buffers through the C-ABI call, copies inside the timed region ----
    lh = torch.from_numpy(left_h).pin_memory().numpy()
    rh = torch.from_numpy(right_h).pin_memory().numpy()
    lab_host = torch.empty((P, cub.y_extent, cub.g_extent), dtype=torch.int32).pin_memory().numpy()
    solver.solve_host(lh[batch(0)], rh[batch(0)], lab_host)
    barrier()
    e2e_ms = []
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        s = batch(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solver.solve_host(lh[s], rh[s], lab_host)   # H2D images, solve, D2H labels
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_value = total_pairs / (max_over_ranks(sum(e2e_ms), world, dev) / 1000.0)

    # ---- roofline of the solve kernel ----
    S = state_bytes(cub.y_extent, cub.g_extent, LABELS)
    upd = [update_bytes(st, cub.y_extent, cub.g_extent, LABELS) for st in all_stats]
    oth = [other_bytes(st, cub.y_extent, cub.g_extent, LABELS) for st in all_stats]
    kern_ms = [st["device_ms"] for st in all_stats]
    # one kernel launch per step solves the whole batch (batched teams), so the
    # step's device time is the kernel's; achieved = node-update bytes / time
    dev_s = sum(step_ms) / 1000.0
    achieved = sum(upd) / dev_s / 1e9
    gnups = sum(st["node_updates"] for st in all_stats) / dev_s / 1e9
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        peak, peak_src = float(json.loads(peaks_path.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    l2 = None
    l2_path = ROOT / "profiles" / "l2_peak.json"
    if l2_path.exists():
        l2_peak = float(json.loads(l2_path.read_text())["l2_read_gbs"])
        l2 = {"peak": l2_peak, "achieved": achieved, "frac": achieved / l2_peak, "unit": "GB/s",
              "peak_source": "profiles/l2_peak.json (tools/micro/l2_bench.cu, measured)"}
    traffic = None
    tr_path = ROOT / "profiles" / "traffic.json"
    if tr_path.exists():
        traffic = json.loads(tr_path.read_text()).get("dram_bytes_per_pair")   # from the committed ncu capture

    # ---- lone-pair latency (the metric's ms per pair): C1 seeds 0-7, one at a time on all SMs ----
    lone = []
    if not args.no_lone:
        for sd in range(8):
            sc = gz.make_scene(sd, W_IMG, H_IMG, DIS_MIN, DIS_MAX)
            vol = gz.sad_volume_device(sc.left, sc.right, cub)
            gz.solve_exact(vol, params)   # warm-up of the lone instance
            lone.append(gz.solve_exact(vol, params).stats["device_ms"])

    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "ms_per_pair": max_ms / (P * args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (make_scene seeds, bit-identical to the reference generator)",
        "config": {"workload": "C4-shaped: batches of Tsukuba 384x288x16 pairs, exact solve (sad_volume + "
                               "solve_exact) per pair; batched teams of GZ_PAIR_TEAM CTAs in one launch",
                   "pairs_per_rank_per_step": P, "image": f"{W_IMG}x{H_IMG}x3", "labels": LABELS,
                   "penalty": PENALTY, "inhibit": INHIBIT, "parallelism": f"pair-sharded x{world}",
                   "l2": "256 MiB buffer written between timed steps (L2 flush)"},
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": int(lh[batch(0)].nbytes * 2),
                "d2h_bytes_per_step": int(lab_host.nbytes)},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "gz4::gz_pairs_kernel (one launch per step, batched teams)",
                     "peak_source": peak_src,
                     "achieved_definition": "SURVEY 8(d): device node_updates x 2S/N_int bytes / step device time",
                     "bytes_per_node_update": 2 * S / (cub.y_extent * cub.g_extent * (LABELS - 1)),
                     "node_update_bytes_per_pair": statistics.mean(upd), "state_bytes_S": S,
                     "other_bytes_per_pair": statistics.mean(oth),
                     "other_bytes_note": "mask builds, BFS levels, reach passes (DESIGN.md section 4); not in achieved",
                     "l2": l2,
                     "limiter": "latency: dependent L2/HBM round trips per group update and per BFS tile round "
                                "(ncu: profiles/)",
                     "mean_pair_device_ms": statistics.mean(kern_ms)},
        "lone_pair_ms": ({"seeds": "0-7", "mean": statistics.mean(lone), "min": min(lone), "max": max(lone),
                          "each": [round(x, 3) for x in lone], "note": "one pair at a time on all SMs (solve_exact)"}
                         if lone else None),
        "gnups": gnups,
        "clocks": clocks.summary(),
        "wall_s_timed_region": wall_s,
        "solver_stats_mean": {k: statistics.mean(st[k] for st in all_stats)
                              for k in ("sweeps", "pulses", "bfs_passes", "reach_passes", "node_updates", "device_ms")},
        "phase_ms_mean": {k: statistics.mean(st["phase_ms"][k] for st in all_stats) for k in all_stats[0]["phase_ms"]},
        "build": _lib.lib().gz_build_info().decode(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n = min(host_threads(), args.cpu_threads)
        rate, wall, flows = cpu_baseline_sample(n, seeds)
        # the same pairs on the device: the baseline's flows double as a parity check
        _, gst = solver.solve(left_d[:n], right_d[:n])
        gflows = [st["flow"] for st in gst]
        if gflows != flows:
            raise SystemExit(f"parity failure: device flows {gflows} != oracle flows {flows}")
        line["cpu_baseline"] = {"value": rate, "unit": "pairs/s", "cores": n, "kind": "port",
                                "sample": f"{n} C1 pairs, one per host thread, {wall:.1f} s wall "
                                          "(oracle/gz_oracle.c: sad_volume + solve_exact)",
                                "parity": f"{n}/{n} device flows equal the oracle's"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
