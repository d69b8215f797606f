"""Summarise an ncu report (+ optional launch-list csv) into a markdown file under profiles/.

python tools/profile_summary.py REP.ncu-rep OUT.md [launches.csv] [title]"""
import collections, csv, io, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3].endswith(".csv") else None
title = sys.argv[-1] if len(sys.argv) > 3 and not sys.argv[-1].endswith(".csv") else rep

def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, rows = raw[0], raw[1], raw[2:]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg"]
lines = [f"# {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none --import-source on)", "",
         "| metric | value | unit |", "|---|---|---|"]
for r in rows[:1]:
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"| {k} | {r[i]} | {units[i]} |")
# dram traffic per launch
try:
    r = rows[0]
    def val(k):
        i = hdr.index(k); v = float(r[i].replace(",", "")); u = units[i]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    lines += ["", f"DRAM traffic per launch (read + write): {(val('dram__bytes_read.sum') + val('dram__bytes_write.sum')) / 1e6:.1f} MB",
              f"L2 sectors per launch (read + write + atom): "
              f"{(val('lts__t_sectors_srcunit_tex_op_read.sum') + val('lts__t_sectors_srcunit_tex_op_write.sum') + val('lts__t_sectors_srcunit_tex_op_atom.sum')) * 32 / 1e9:.2f} GB"]
except Exception as ex:  # noqa
    lines.append(f"(traffic summary unavailable: {ex})")
# per-source-line stall samples
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
agg = collections.Counter(); text = {}; fname = None; si = None; line = None
for r in src:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)"); continue
    if si is None or len(r) <= si:
        continue
    if r[0]:
        line = (fname, int(r[0])); text[line] = r[1].strip()[:90]
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if line:
        agg[line] += v
tot = sum(agg.values()) or 1
lines += ["", "## Warp-stall samples by source line (top 25)", "", "| share | line | source |", "|---|---|---|"]
for (f, l), v in agg.most_common(25):
    lines.append(f"| {100 * v / tot:.1f}% | {f}:{l} | `{text.get((f, l), '').replace('|', '/')}` |")
if launches:
    rows = list(csv.reader(open(launches)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]; ki, vi = H.index("Kernel Name"), H.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    lines += ["", f"## Launch list (`{launches}`, gpu__time_duration, cold-cache serialised)", "",
              "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
open(out, "w").write("\n".join(lines) + "\n")
print("wrote", out)
