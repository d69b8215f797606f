"""Per-source-line totals of an ncu report: instructions executed, L2 sectors
(global), stall samples -- which source lines the kernel's work comes from.

python tools/ncu_lines.py REP.ncu-rep [top]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout)))
cols = {}
agg = {k: collections.Counter() for k in ("inst", "l2", "stall")}
text, fname, line = {}, None, None
for r in src:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        cols = {"inst": r.index("Instructions Executed"), "l2": r.index("L2 Theoretical Sectors Global"),
                "stall": r.index("Warp Stall Sampling (All Samples)")}
        continue
    if not cols or len(r) <= max(cols.values()):
        continue
    if r[0]:
        line = (fname, int(r[0]))
        text[line] = r[1].strip()[:80]
        for k, i in cols.items():   # the cuda line rows carry the per-line totals
            try:
                agg[k][line] += float(r[i] or 0)
            except ValueError:
                pass
for k in ("inst", "l2", "stall"):
    tot = sum(agg[k].values()) or 1
    print(f"\n== {k}: total {tot:.3e}")
    for (f, l), v in agg[k].most_common(top):
        print(f"{100 * v / tot:5.1f}%  {f}:{l}  {text.get((f, l), '')}")
