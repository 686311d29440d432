"""Per-source-line warp-level instructions executed (column 'Instructions Executed')
from an `ncu --page source --csv --print-source cuda,sass` export.
usage: python tools/ncu_inst_lines.py mix.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur = (f, r[0], r[1].strip()[:70])
        continue
    try:
        agg[cur] = agg.get(cur, 0.0) + float(r[ix] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(agg.values()) or 1.0
print(f"total warp instructions {tot:.3e}")
for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln} {src}")
