"""Per-pulse trace of lone C1 solves (GZ_TRACE=2): time spent in pulses by
active-group count, to see where a lone solve's ~450 pulses go.

python tools/lone_trace.py SEED [SEED ...]   (run under gpurun)"""
import collections, os, re, subprocess, sys
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
code = f"""
import sys; sys.path.insert(0, {ROOT!r})
import paper_1803_01516_b200 as gz
cub = gz.cuboid_from_disparity_range(384, 288, 10, 28, num_labels=16)
sc = gz.make_scene(int(sys.argv[1]))
vol = gz.sad_volume_device(sc.left, sc.right, cub)
gz.solve_exact(vol, gz.EnergyParams(14, 1023))
import os; os.environ['GZ_TRACE'] = '2'
r = gz.solve_exact(vol, gz.EnergyParams(14, 1023))
print('device_ms', r.stats['device_ms'], 'pulses', r.stats['pulses'], r.stats['phase_ms'])
"""
for seed in sys.argv[1:]:
    p = subprocess.run([sys.executable, "-c", code, seed], capture_output=True, text=True)
    print(f"seed {seed}:", p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-500:])
    raw = [l for l in p.stderr.splitlines() if l.startswith("gz_pulse")]
    open(os.path.join(ROOT, "gpurun_out", f"lone_trace_{seed}.raw"), "w").write("\n".join(raw) + "\n")
    tail = collections.defaultdict(lambda: [0, 0.0, 0])
    for line in raw:
        m = re.match(r"gz_pulse sweep (\d+) pulse (\d+) groups (\d+) dt_us ([\d.]+)", line)
        if m and int(m.group(2)) >= 1000:
            t = tail[int(m.group(1))]
            t[0] += 1; t[1] += float(m.group(4)); t[2] += int(m.group(3))
    for sw in sorted(tail):
        n, t, g = tail[sw]
        print(f"  sweep {sw:3d} tail: {n:3d} pulses, {t / 1000:6.3f} ms, {g / max(n, 1):6.1f} groups/pulse")
    buckets = collections.defaultdict(lambda: [0, 0.0, 0])
    for line in p.stderr.splitlines():
        m = re.match(r"gz_pulse sweep (\d+) pulse (\d+) groups (\d+) dt_us ([\d.]+)", line)
        if not m:
            continue
        g, dt = int(m.group(3)), float(m.group(4))
        if int(m.group(2)) >= 1000:
            continue
        b = 0 if g == 0 else 1 if g <= 8 else 2 if g <= 64 else 3 if g <= 512 else 4 if g <= 4096 else 5
        buckets[b][0] += 1
        buckets[b][1] += dt
        buckets[b][2] += g
    names = ["0", "1-8", "9-64", "65-512", "513-4096", ">4096"]
    for b in sorted(buckets):
        n, t, g = buckets[b]
        print(f"  groups {names[b]:>9s}: {n:4d} pulses, {t / 1000:7.3f} ms, {t / max(n, 1):6.2f} us/pulse, {g} groups")
