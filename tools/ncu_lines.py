"""Aggregate ncu warp-stall samples per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [top]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.Counter(); src = {}
fname = None; hdr = None; line = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if r[0] == 'Line No':
        hdr = r; si = r.index('Warp Stall Sampling (All Samples)'); continue
    if hdr is None or len(r) <= si:
        continue
    if r[0]:
        line = (fname, int(r[0])); src[line] = r[1][:100]
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    if line:
        agg[line] += v
tot = sum(agg.values())
print("total samples", tot)
for (f, l), v in agg.most_common(top):
    print(f"{100*v/tot:5.1f}% {f}:{l}  {src.get((f,l),'')}")
